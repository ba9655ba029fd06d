"""The seeded input generators: deterministic, slice-consistent, right statistics."""
import numpy as np

import synth


def test_uniform_deterministic_and_sliceable():
    a = synth.uniform_f32(123, 1000)
    b = synth.uniform_f32(123, 400, off=300)
    np.testing.assert_array_equal(a[300:700], b)
    assert a.min() >= 0.0 and a.max() < 1.0
    assert abs(a.mean() - 0.5) < 0.05
    # on the 2^-24 grid
    np.testing.assert_array_equal(a * 2 ** 24, np.floor(a * 2 ** 24))


def test_f16grid_exact_in_fp16():
    a = synth.uniform_f16grid(5, 5000)
    np.testing.assert_array_equal(a.astype(np.float16).astype(np.float32), a)


def test_normal_moments():
    a = synth.normal_f32(9, 200000)
    assert abs(a.mean()) < 0.02 and abs(a.std() - 1.0) < 0.02


def test_config_rows_and_batch_slices_match_full():
    cfg = synth.CONFIGS["C3"]
    full = synth.make_values(cfg, 0, 2)
    rows = synth.make_values(cfg, 0, 2, rows=(17, 60))
    np.testing.assert_array_equal(full[:, :, 17:60], rows)
    sl = synth.make_values(cfg, 1, 2)
    np.testing.assert_array_equal(full[1:2], sl)


def test_field_rows_match():
    a = synth.field_f32(77, 256, 256, 0, 256)
    b = synth.field_f32(77, 256, 256, 100, 140)
    np.testing.assert_array_equal(a[100:140], b)
    assert np.abs(a).max() < 1.02
    # smooth: neighbouring pixels differ far less than the value range
    assert np.abs(np.diff(a, axis=1)).mean() < 0.1 * (a.max() - a.min())
