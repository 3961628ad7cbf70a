"""Input generator: deterministic, chunk-order independent, paper sizes (CPU)."""
import os

import numpy as np

from synth import CONFIGS, cars, generate, reference


def test_sizes():
    assert CONFIGS["cfg1"].n_pixels == 4096 and CONFIGS["cfg2"].n_pixels == 65536
    assert CONFIGS["cfg3"].n_pixels == 703026 and CONFIGS["cfg4"].n_pixels == 4_000_000
    assert CONFIGS["cfg5_apply"].n_pixels == 703026


def test_deterministic_and_chunk_independent():
    cfg = CONFIGS["cfg2"].with_(height=300, width=300, n_freq=64)   # 90,000 rows -> 2 blocks
    a, ra, _ = generate(cfg, threads=1)
    b, rb, _ = generate(cfg, threads=4)
    assert a.dtype == np.float32 and np.array_equal(a, b) and np.array_equal(ra, rb)
    # the second block does not depend on the first
    inst = cars.instrument(cfg)
    conc = cars.concentrations(cfg)
    out = np.zeros_like(a)
    cars._block(cfg, inst, conc, 1, out, np.float32)
    assert np.array_equal(out[cars.BLOCK_ROWS:], a[cars.BLOCK_ROWS:])


def test_reference_positive_and_instrument_shared():
    r5t = reference(CONFIGS["cfg5_train"])
    r5a = reference(CONFIGS["cfg5_apply"])
    assert np.all(r5t > 0) and np.array_equal(r5t, r5a)     # same instrument (species_seed 1)
    assert np.all(reference(CONFIGS["cfg3"]) > 0)


def test_paper_simulation_sizes_and_physics():
    """synth.paper_simulation follows PAPER.md:194: side-scaled sizes (P19 totals), noiseless
    I = |chi|^2, Raman peaks only in 500-1700 cm^-1 (Im{chi/chi_nr} ~ 0 far outside), a positive real
    linear reference."""
    import json
    from synth.cars import paper_sim_shape, paper_simulation
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
    for sc, tot in zip(gold["sim_side_scaled_totals"]["scales"], gold["sim_side_scaled_totals"]["value"]):
        h, w = paper_sim_shape(sc)
        assert h * w == tot
    I, Iref, truth, om = paper_simulation(0.5)
    assert I.shape == (4551, 812) and np.all(I > 0) and np.all(Iref > 0)
    far = (om < 300) | (om > 1900)
    assert np.max(np.abs(truth[:, far])) < 0.1 * np.max(np.abs(truth))
    assert np.all(np.diff(Iref.astype(np.float64)) >= 0) or np.all(np.diff(Iref.astype(np.float64)) <= 0)
