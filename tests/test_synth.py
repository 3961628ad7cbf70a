"""Input generator: deterministic, chunk-order independent, paper sizes (CPU)."""
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
