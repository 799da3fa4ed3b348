"""Pins for the shared seeded input generator (graf_inputs)."""
import numpy as np

from graf_inputs import (CONFIGS, SplitMix64, barker13, config_waveforms, frank,
                         p4, waveform)


def test_splitmix64_reference_vector():
    # Published splitmix64 outputs for seed 0 (Vigna's reference C code).
    r = SplitMix64(0)
    assert [int(x) for x in r.u64(4)] == [
        0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]


def test_stream_is_counter_based():
    a = SplitMix64(7)
    x = np.concatenate([a.u64(3), a.u64(5)])
    assert np.array_equal(x, SplitMix64(7).u64(8))


def test_uniform_and_gaussian_moments():
    r = SplitMix64(123)
    u = r.uniform(200000)
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 5e-3
    z = SplitMix64(321).gaussian(200000)
    assert abs(z.mean()) < 1e-2 and abs(z.std() - 1) < 1e-2


def test_config_shapes_and_families():
    for c, cfg in CONFIGS.items():
        s = config_waveforms(c, batch=2, n=min(cfg["N"], 256) if c != 3 else None)
        assert s.dtype == np.complex64 and s.shape[0] == 2
    # c1 waveform is seed 0 and unimodular
    s1 = waveform(1, 0)
    assert s1.shape == (64,) and np.allclose(np.abs(s1), 1, atol=1e-6)
    # c3 families: LFM / Frank|P4 / QPSK, all unimodular
    s3 = config_waveforms(3, batch=6)
    assert np.allclose(np.abs(s3), 1, atol=1e-6)
    assert np.array_equal(s3[1], frank(1024)) and np.array_equal(s3[4], p4(1024))
    q = s3[2]
    assert set(np.round(q.real).astype(int) + 10 * np.round(q.imag).astype(int)) <= {1, -1, 10, -10}
    # c4: ripple sigma 0.05 around unit amplitude
    a = np.abs(waveform(4, 0))
    assert abs(a.mean() - 1) < 5e-3 and abs(a.std() - 0.05) < 5e-3


def test_barker13_values():
    b = barker13()
    assert b.shape == (13,) and np.array_equal(np.abs(b), np.ones(13, np.float32))
