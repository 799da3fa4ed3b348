"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and rejects malformed arguments on the host before any CUDA
call (include/graf.h 'Errors')."""
import ctypes
import os
import re

import pytest

from paper_2506_22935_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "graf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(graf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    names = header_functions()
    assert set(L.EXPORTS) == set(names), names
    for n in names:
        assert hasattr(lib, n), n
    assert lib.graf_abi_version() == L.ABI_VERSION


def test_status_strings():
    lib = L.lib()
    for st in range(6):
        assert lib.graf_status_string(st).decode().startswith("GRAF_")


def desc(n=64, m=64, b=1, out=L.OUT_NONE, kb=None, ke=None, shard=(0, 1), ver=L.ABI_VERSION):
    return L.AfDesc(ver, n, m, out, b, -(n - 1) if kb is None else kb, n if ke is None else ke,
                    L.DOPPLER_CENTERED, 0, shard[0], shard[1])


def loss(kmax=8, dmax=8, mlk=0, mld=0, lpsl=0.0, T=0.01, norm=1):
    return L.LossDesc(kmax, dmax, mlk, mld, None, None, 1.0, lpsl, T, norm)


FAKE = ctypes.c_void_p(1 << 20)   # never dereferenced: every case fails validation first


@pytest.mark.parametrize("d,ld,expect", [
    (desc(ver=99), loss(), L.GRAF_EINVAL),
    (desc(n=0), loss(), L.GRAF_EINVAL),
    (desc(b=0), loss(), L.GRAF_EINVAL),
    (desc(m=48), loss(), L.GRAF_EINVAL),
    (desc(n=64, m=32), loss(), L.GRAF_EUNSUPPORTED),
    (desc(n=20000, m=32768), loss(), L.GRAF_EUNSUPPORTED),
    (desc(shard=(2, 2)), loss(), L.GRAF_EINVAL),
    (desc(), loss(kmax=0, dmax=0), L.GRAF_EINVAL),          # empty region
    (desc(), loss(kmax=-1), L.GRAF_EINVAL),
    (desc(), loss(lpsl=1.0, T=0.0), L.GRAF_EINVAL),
    (desc(), loss(norm=3), L.GRAF_EINVAL),
])
def test_loss_grad_rejects(d, ld, expect):
    lib = L.lib()
    st = lib.graf_af_loss_grad(ctypes.byref(d), ctypes.byref(ld), FAKE, None, None, FAKE, None, FAKE,
                               1 << 30, None)
    assert st == expect, lib.graf_last_error()
    assert lib.graf_last_error().decode()


def test_forward_rejects_bad_window_and_surface():
    lib = L.lib()
    d = desc(out=L.OUT_ABS_F32, kb=-64, ke=3)
    assert lib.graf_af_forward(ctypes.byref(d), None, FAKE, FAKE, None, FAKE, 1 << 30, None) == L.GRAF_EINVAL
    d = desc(out=L.OUT_ABS_F32)
    assert lib.graf_af_forward(ctypes.byref(d), None, FAKE, None, None, FAKE, 1 << 30, None) == L.GRAF_EINVAL
    d = desc(out=L.OUT_C64)
    mis = ctypes.c_void_p((1 << 20) + 4)
    assert lib.graf_af_forward(ctypes.byref(d), None, mis, FAKE, None, FAKE, 1 << 30, None) == L.GRAF_EINVAL


def test_workspace_check_and_size():
    lib = L.lib()
    d = desc(n=256, m=256, b=256)
    ld = loss(kmax=64, dmax=32)
    need = lib.graf_workspace_bytes(ctypes.byref(d), ctypes.byref(ld))
    assert need > 0 and need % 256 == 0
    st = lib.graf_af_loss_grad(ctypes.byref(d), ctypes.byref(ld), FAKE, None, None, FAKE, None, FAKE,
                               256, None)
    assert st == L.GRAF_EWORKSPACE
    assert lib.graf_workspace_bytes(ctypes.byref(desc(n=0)), None) == 0


def test_backward_rejects():
    lib = L.lib()
    d = desc()
    assert lib.graf_af_backward(ctypes.byref(d), FAKE, None, FAKE, FAKE, 1 << 30, None) == L.GRAF_EINVAL
    d = desc(kb=5, ke=5)
    assert lib.graf_af_backward(ctypes.byref(d), FAKE, FAKE, FAKE, FAKE, 1 << 30, None) == L.GRAF_EINVAL


def test_host_combine_partials_is_exact_lse_merge():
    import math
    lib = L.lib()
    T = 0.5
    ld = L.LossDesc(1, 1, 0, 0, None, None, 1.0, 1.0, T, 1, 0.0, 0.0, None, 0)
    # two shards, one waveform: shard sums of exp((x-m)/T) over {0.1, 0.3} and {0.7}
    sh = (L.Partials * 2)(L.Partials(1.0, 0.3, math.exp((0.1 - 0.3) / T) + 1.0, 0.0, 7.0, 0.0),
                          L.Partials(2.0, 0.7, 1.0, 0.0, 5.0, 0.0))
    out = L.Partials()
    assert lib.graf_combine_partials(ctypes.byref(ld), sh, 2, 1, ctypes.byref(out), 0, None) == L.GRAF_OK
    ref = sum(math.exp((x - 0.7) / T) for x in (0.1, 0.3, 0.7))
    assert out.isl_sum == 3.0 and abs(out.lse_max - 0.7) < 1e-7 and abs(out.lse_sum - ref) < 1e-6
    assert out.psl_key == 5.0                      # the argmax cell of the larger max


# The launch model (choose_P, csrc/graf_launch.cuh).  Expected values
# are the CTAs per waveform measured fastest on one B200 (profiles/r01_p_sweep.txt for the
# full batches, profiles/r02/shard/p_variants_*.txt for the batch-sharded blocks):
# (rows, slots, batch, resident CTAs per SM, P bound) -> P.
@pytest.mark.parametrize("rows,slots,batch,occ,p_bound,expect", [
    (65, 8, 256, 4, 5, 2),          # c2 (fused cluster finalize, P = 2)
    (1024, 4, 1024, 2, 2, 2),       # c3
    (1024, 4, 512, 2, 3, 2),        # c3 half batch: the plain wave model ties P = 1 (slower)
    (513, 1, 64, 2, 19, 9),         # c4
    (513, 1, 16, 2, 74, 18),        # c4 block of 16: needs occ = 2 (the API reported 1 -> P = 9)
    (513, 1, 8, 2, 148, 37),        # c4 block of 8
    (16384, 1, 8, 1, 148, 37),      # c5: 296 CTAs, two waves of one CTA per SM
    (2048, 1, 8, 1, 148, 37),       # c5, one shard of G = 8
])
def test_launch_model_ctas_per_waveform(rows, slots, batch, occ, p_bound, expect):
    lib = L.lib()
    assert lib.graf_plan_ctas_per_waveform(rows, slots, batch, occ, 148, p_bound) == expect


def test_launch_model_bounds_and_bad_arguments():
    lib = L.lib()
    for args in [(0, 1, 1, 1, 148, 1), (1, 0, 1, 1, 148, 1), (1, 1, 0, 1, 148, 1), (1, 1, 1, 0, 148, 1),
                 (1, 1, 1, 1, 0, 1), (1, 1, 1, 1, 148, 0)]:
        assert lib.graf_plan_ctas_per_waveform(*args) == 0
    for rows, slots, batch, occ, pb in [(1, 16, 1, 4, 8), (64, 16, 1, 4, 4), (4095, 2, 3, 2, 400), (513, 1, 64, 2, 1)]:
        p = lib.graf_plan_ctas_per_waveform(rows, slots, batch, occ, 148, pb)
        assert 1 <= p <= pb
