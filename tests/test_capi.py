"""CPU-side checks of the product boundary (no GPU needed):
the C-ABI library loads and exports every symbol include/fcwave_b200.h
declares, the host geometry is integer-exact against the oracle, the error
classes mirror the reference's exceptions, and the product package never
imports the oracle."""
import ast
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2008_00672_b200 as fb
from paper_2008_00672_b200 import _lib, configs
from paper_2008_00672_b200 import fcwave as fc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fcwave_b200.h")).read()
    return sorted(set(re.findall(r"\b(fcw_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTS) == syms
    assert L.fcw_version().decode().startswith("fcwave-b200")


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2008_00672_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert not (node.module or "").startswith("oracle"), f


def test_geometry_matches_oracle():
    for scs, n in [(15, 1024), (15, 2048), (15, 512), (30, 4096)]:
        assert fc.cp_schedule(scs, n, 14) == O.cp_schedule(scs, n, 14)
    for N, L, lam in [(1024, 128, 0.5), (1024, 16, 0.5), (1024, 128, 0.25), (4096, 256, 0.5), (32, 8, 0.5)]:
        a, b = fb.derive_fc_params(N, L, lam), O.derive_params(N, L, lam)
        assert a.__dict__ == b.__dict__
    for ncp in (72, 80, 144, 160, 288, 352):
        for I in (1, 4, 8, 16, 64, 256):
            assert fb.cp_truncate(ncp, I) == O.cp_truncate(ncp, I)
    for L, npass, ntb in [(16, 12, 2), (512, 288, 4), (256, 144, 4), (32, 8, 1)]:
        assert np.array_equal(fb.design_window(L, npass, ntb), O.design_window(L, npass, ntb))
    for l, na, sk in [(16, 12, False), (16, 8, True), (512, 408, False), (256, 144, False)]:
        assert fb.centered_active_map(l, na, sk) == O.centered_active_map(l, na, sk)
    cps = fb.CpSchedule([80, 72, 72, 72])
    p = fb.derive_fc_params(1024, 16)
    for n in range(4):
        assert fb.symbol_sigma(n, cps, 1024) == O.symbol_sigma(n, cps.per_symbol_high_rate, 1024)
    assert fb.combined_length(4, cps, p) == O.combined_length(4, cps.per_symbol_high_rate, O.derive_params(1024, 16))
    assert fb.first_block_overlap(fb.derive_fc_params(1024, 128), 9) == pytest.approx(0.4296875, abs=1e-12)
    assert fb.first_block_overlap(fb.derive_fc_params(64, 16), 1) == pytest.approx(0.4375, abs=1e-12)


def test_nr_cp_schedule():
    s = fb.nr_cp_schedule(fb.make_numerology(30, 4096), 28).per_symbol_high_rate
    assert s[0] == 352 and s[14] == 352 and all(v == 288 for i, v in enumerate(s) if i not in (0, 14))
    assert sum(s[:14]) + 14 * 4096 == 61440  # 0.5 ms at 122.88 Msps
    assert fb.nr_cp_schedule(fb.make_numerology(15, 1024), 14).per_symbol_high_rate == O.cp_schedule(15, 1024, 14)
    assert fb.nr_cp_schedule(fb.make_numerology(15, 2048), 14).per_symbol_high_rate == O.cp_schedule(15, 2048, 14)


def test_error_classes_mirror_reference():
    with pytest.raises(ValueError):
        fb.derive_fc_params(1024, 96, 0.5)
    with pytest.raises(ValueError):
        fb.design_window(16, 14, 2)
    with pytest.raises(ValueError):
        fb.centered_active_map(16, 16)
    with pytest.raises(ValueError):
        fb.make_numerology(15, 100)
    with pytest.raises(ValueError):
        fb.first_block_overlap(fb.derive_fc_params(64, 16), 5)
    with pytest.raises(ValueError):
        fc.cp_schedule(15, 16, 7)


def _plan_args(N, cps, subs):
    arr = (_lib.SubbandC * len(subs))()
    keep = []
    for m, (L, c, lofdm, w, bins) in enumerate(subs):
        b = np.asarray(bins, np.int32)
        wd = np.asarray(w, np.float64)
        keep += [b, wd]
        arr[m].L, arr[m].l_ofdm, arr[m].c, arr[m].n_active = L, lofdm, c, len(b)
        arr[m].active_bins = b.ctypes.data_as(C.POINTER(C.c_int))
        arr[m].window = wd.ctypes.data_as(C.POINTER(C.c_double))
    cp = np.asarray(cps, np.int32)
    keep.append(cp)
    return arr, cp, keep


@pytest.mark.parametrize("N,cps,subs,code", [
    # reference preconditions -> FCW_EINVAL (std::invalid_argument)
    (1024, [80, 72], [(96, 0, 96, np.ones(96), [0])], _lib.FCW_EINVAL),            # L does not divide N
    (1024, [80, 72], [(16, 0, 32, np.ones(16), [0])], _lib.FCW_EINVAL),            # L != L_OFDM
    (1024, [400, 72], [(16, 0, 16, np.ones(16), [0])], _lib.FCW_EINVAL),           # l_cp > L_L
    (1024, [80, 72], [(16, 0, 16, np.ones(16), [16])], _lib.FCW_EINVAL),           # active bin out of [0,L)
    (1024, [80, 72], [(16, 0, 16, np.ones(16), [1, 1])], _lib.FCW_EINVAL),         # duplicate active bin
    # valid for the reference, outside this build's envelope -> FCW_ENOTSUP
    (8192, [80, 72], [(16, 0, 16, np.ones(16), [0])], _lib.FCW_ENOTSUP),           # N > 4096
    (4096, [80, 72], [(2048, 0, 2048, np.ones(2048), [0])], _lib.FCW_ENOTSUP),     # L > 1024
])
def test_plan_validation_codes(N, cps, subs, code):
    arr, cp, keep = _plan_args(N, cps, subs)
    h = C.c_void_p()
    rc = _lib.lib().fcw_plan_create(C.byref(h), N, 0.5, cp.ctypes.data_as(C.POINTER(C.c_int)), len(cps), arr,
                                    len(subs), 0)
    assert rc == code, _lib.lib().fcw_last_error()
    assert not h.value


def test_overlap_other_than_half_is_unsupported_not_silent():
    arr, cp, keep = _plan_args(1024, [80, 72], [(16, 0, 16, np.ones(16), [0])])
    h = C.c_void_p()
    rc = _lib.lib().fcw_plan_create(C.byref(h), 1024, 0.25, cp.ctypes.data_as(C.POINTER(C.c_int)), 2, arr, 1, 0)
    assert rc == _lib.FCW_ENOTSUP


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(fb.FcwError):
        configs.config1().plan()


def test_workload_geometry():
    """BASELINE configs: allocation, Q and frame length are what SURVEY App. A states."""
    c1, c2, c4, c5 = configs.config1(), configs.config2(), configs.config4(), configs.config5()
    assert c1.cp == [80, 72] and c1.subbands[0].L == 16
    assert O.combined_length(2, c1.cp, O.derive_params(1024, 16)) == 2632
    assert [s.L for s in c2.subbands] == [512] * 4 and [len(b) for b in c2.active_maps] == [288, 288, 288, 408]
    assert O.combined_length(14, c2.cp, O.derive_params(2048, 512)) == 31584
    for w in (c4, c5):
        assert O.combined_length(280, w.cp, O.derive_params(4096, w.subbands[0].L)) == 1230496
        assert sum(4096 + c for c in w.cp) == 1228800
        assert sum(len(b) for b in w.active_maps) == 3276
    assert c4.units == 4 and c5.units == 512
    # contiguous allocations: every grid bin carries at most one active subcarrier
    for w in (c2, c4, c5):
        used = []
        for s, bins in zip(w.subbands, w.active_maps):
            for b in bins:
                ls = b if b < s.L // 2 else b - s.L
                used.append((s.c + ls) % w.N)
        assert len(used) == len(set(used))
        assert (max((u + w.N // 2) % w.N for u in used) - min((u + w.N // 2) % w.N for u in used) + 1) == len(used)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_workload_geometry_backends_agree(name):
    """bench.py's reference arm builds every workload from the oracle's geometry
    (no product library loaded); it must be bit-identical to the product's."""
    a, b = configs.get(name), configs.get(name, geom=O.Geometry())
    banks_a = a.banks if hasattr(a, "banks") else [a]
    banks_b = b.banks if hasattr(b, "banks") else [b]
    assert len(banks_a) == len(banks_b)
    for x, y in zip(banks_a, banks_b):
        assert (x.N, x.cp, x.active_maps, x.bits_per_symbol) == (y.N, y.cp, y.active_maps, y.bits_per_symbol)
        for s, t in zip(x.subbands, y.subbands):
            assert (s.L, s.c, s.n_active, s.n_tb, s.l_ofdm) == (t.L, t.c, t.n_active, t.n_tb, t.l_ofdm)
            assert np.array_equal(np.asarray(s.window).view(np.uint64), np.asarray(t.window).view(np.uint64))


def test_nr_cp_schedule_matches_oracle_restatement():
    for scs, n, B in [(30, 4096, 280), (15, 2048, 28), (60, 4096, 60), (30, 1024, 30)]:
        assert fb.nr_cp_schedule(fb.make_numerology(scs, n), B).per_symbol_high_rate == O.nr_cp_schedule(scs, n, B)
    assert O.nr_cp_schedule(30, 4096, 15)[::14] == [352, 352] and O.nr_cp_schedule(30, 4096, 15)[1] == 288


def test_configs_import_without_product_library():
    """Importing the workload definitions with the oracle backend loads no product code."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r); import oracle as O; "
            "from paper_2008_00672_b200 import configs; w = configs.config5(geom=O.Geometry()); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'libfcwave_b200' not in maps, 'product library mapped'; "
            "assert 'paper_2008_00672_b200.api' not in sys.modules; print('ok')" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


def test_symbol_and_block_phase_match_oracle():
    """fcw_symbol_phase / fcw_block_phase (double, host) against the oracle's
    restatement of fc_sync.cpp:45-50 / fc_core.cpp:41-44."""
    rng = np.random.default_rng(3)
    cp = [352] + [288] * 13 + [352] + [288] * 5
    cps = fb.CpSchedule(cp)
    for _ in range(50):
        # c >= 0: bit-exact; c < 0: the reference's truncating % gives the
        # co-terminal angle (-x instead of 2 pi - x), equal to 1e-15
        n, c = int(rng.integers(0, len(cp))), int(rng.integers(-5000, 5000))
        r, L = int(rng.integers(0, 3)), int(2 ** rng.integers(2, 11))
        a, b = fb.symbol_phase(n, c, cps, 4096), O.symbol_phase(n, c, cp, 4096)
        e, f = fb.block_phase(r, c, L // 2, L), O.block_phase(r, c, L // 2, L)
        if c >= 0:
            assert a == b and e == f
        assert abs(a - b) < 1e-15 and abs(e - f) < 1e-15
    with pytest.raises(ValueError):
        fb.symbol_phase(-1, 3, cps, 4096)
