"""Seeded synthetic CARS inputs (no method arithmetic); see synth/cars.py."""
from .cars import (BLOCK_ROWS, CONFIGS, CubeConfig, concentrations, generate, generate_rows, instrument,
                   lorentzian_spectrum, omega_axis, reference, truth_imag)

__all__ = ["BLOCK_ROWS", "CONFIGS", "CubeConfig", "concentrations", "generate", "generate_rows", "instrument",
           "lorentzian_spectrum", "omega_axis", "reference", "truth_imag"]
