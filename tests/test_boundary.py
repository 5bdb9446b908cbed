"""The C-ABI boundary: libsht.so builds, loads, exports every symbol of
include/sht.h, and its host-only helpers agree with the oracle bit for bit.
No GPU compute is called here."""

import json
import re
from pathlib import Path

import numpy as np
import pytest

from oracle.sht_oracle import gauss_nodes as oracle_nodes
from oracle.transposition import Layout, ring_fft_cost, ring_partition, snake
from oracle.sht_oracle import SHTransformOracle

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "sht.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sht_\w+)\s*\(", text, re.M)))


def test_exports_every_header_symbol(lib):
    from paper_1908_06097_b200 import _lib

    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms
    assert lib.sht_version() >= 100


def test_library_is_sm100a(lib):
    import subprocess

    from paper_1908_06097_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass            # FP64 tensor-core Legendre GEMMs
    assert "LDGSTS" in sass                # cp.async operand staging


@pytest.mark.parametrize("ndgl", [2, 160, 1280, 2560])
def test_gauss_nodes_bit_identical(lib, ndgl):
    from paper_1908_06097_b200 import gauss_nodes

    a = gauss_nodes(ndgl)
    b = oracle_nodes(ndgl)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("T,P", [(79, 1), (79, 2), (639, 4), (639, 8), (20, 3)])
def test_partition_matches_restatement(lib, T, P):
    from paper_1908_06097_b200 import partition

    mo, ro = partition(T, P)
    nloen = 4 * np.arange(1, T + 2) + 16
    mc = np.minimum(T, (nloen - 1) // 2)
    assert np.array_equal(mo, snake(T + 1, P))
    assert np.array_equal(ro, ring_partition(nloen, mc, P))
    # balance at TCo639: Legendre work within 2%, ring-FFT cost within 0.1%, grid points within 5%
    if T == 639:
        ndglu = np.array([(mc >= m).sum() for m in range(T + 1)])
        work = ndglu * (T - np.arange(T + 1) + 1)
        wr = np.bincount(mo, weights=work, minlength=P)
        cost = np.array([ring_fft_cost(int(n), int(m)) for n, m in zip(nloen, mc)])
        cr = np.bincount(ro, weights=cost, minlength=P)
        pr = np.bincount(ro, weights=nloen, minlength=P)
        assert wr.max() / wr.mean() < 1.02 and cr.max() / cr.mean() < 1.001 and pr.max() / pr.mean() < 1.05


@pytest.mark.parametrize("T,P", [(15, 2), (79, 3), (639, 8)])
def test_alltoall_rows_match_restatement(lib, T, P):
    from paper_1908_06097_b200 import alltoall_rows

    o = SHTransformOracle(T, nfld=1) if T < 100 else None
    rows = alltoall_rows(T, P)
    if o is not None:
        assert np.array_equal(rows, Layout(o, P).rows())
    nloen = 4 * np.arange(1, T + 2) + 16
    assert rows.sum() == int(np.sum(np.minimum(T, (nloen - 1) // 2) + 1))   # every (ring pair, m) once


def test_alltoall_order_is_reference_rotated_schedule(lib):
    """Issue order == haloflow build_alltoall(ROTATED_CONCURRENT) (collectives.py:85-86),
    pinned by tests/golden/schedules.json generated from the reference itself."""
    from paper_1908_06097_b200 import alltoall_order

    gold = json.loads((ROOT / "tests" / "golden" / "schedules.json").read_text())["rotated_order"]
    for P, flows in gold.items():
        P = int(P)
        ours = [[r, d] for r in range(P) for d in alltoall_order(P, r)]
        assert ours == flows


def test_size_matrix_golden(lib):
    from paper_1908_06097_b200 import alltoall_rows

    gold = json.loads((ROOT / "tests" / "golden" / "schedules.json").read_text())["tco639"]
    for P, d in gold.items():
        assert alltoall_rows(639, int(P)).tolist() == d["rows"]
        ms = d["makespan_s"]
        assert ms["rotated_concurrent"] <= min(ms.values()) + 1e-12   # the paper's winner


def test_bluestein_length_matches_restatement(lib):
    """libsht's cost-chosen whole-ring Bluestein lengths == the restatement used by the partition model."""
    from oracle.transposition import _bluestein_len, _factor
    from paper_1908_06097_b200 import fft_plan_info

    checked = 0
    for n in range(20, 2600, 4):
        info = fft_plan_info(n)            # no pruning: |k| <= n/2 kept
        primes, _ = _factor(n, n)
        if not (any(p > 127 for p in primes) or sum(p > 16 for p in primes) >= 2):
            continue                       # direct, possibly with a DMMA prime step
        L, rad = _bluestein_len(2 * n - 1, 6022)
        if L < 0:
            L, rad = _bluestein_len(2 * n - 1, 12288)
        if 0 < L <= 12288:
            assert info["length"] == L and info["radices"] == rad, n
            checked += 1
    assert checked > 100


def test_fft_plans(lib):
    from paper_1908_06097_b200 import fft_plan_info

    p20 = fft_plan_info(20)
    assert p20["length"] == 20 and not p20["bluestein"] and len(p20["radices"]) == 2
    assert len(fft_plan_info(2560)["radices"]) == 3                 # 16 x 16 x 10
    assert not fft_plan_info(2576)["bluestein"]                     # 2^4 * 7 * 23: direct, DMMA prime-23 step
    assert fft_plan_info(2576)["radices"][-1] == 23
    p508 = fft_plan_info(508)                                       # 4 * 127: the largest DMMA prime step
    assert not p508["bluestein"] and p508["radices"] == [4, 127]

    big = fft_plan_info(2572)                                       # 4 * 643: whole-ring Bluestein
    assert big["bluestein"] and big["length"] >= 2 * 2572 - 1
    assert fft_plan_info(8016)["radices"][-1] == 167                # factor-local Bluestein step (TCo1999)
    assert fft_plan_info(6364)["radices"][-2:] == [37, 43]          # two Bluestein steps (TCo1999 ring)
    assert fft_plan_info(5476)["length"] == 11264                   # 4 * 37^2: whole-ring Bluestein, 212 KB class
    for n in list(range(20, 2600, 4)) + list(range(2600, 8020, 52)):   # TCo639 .. TCo1999 rings
        info = fft_plan_info(n)
        assert int(np.prod(info["radices"])) == info["length"]
        if info["length"] != n:                                     # whole-ring Bluestein
            assert info["bluestein"] and info["length"] >= 2 * n - 1
        elif not info["bluestein"]:                                 # direct: <= one DMMA prime step, last
            big = [r for r in info["radices"] if r > 16]
            assert len(big) <= 1 and all(r <= 127 for r in big) and (not big or info["radices"][-1] == big[0])


def test_errors_map_to_reference_classes(lib):
    from paper_1908_06097_b200 import ConfigurationError, alltoall_order, partition

    with pytest.raises(ConfigurationError):
        partition(0, 2)
    with pytest.raises(ConfigurationError):
        partition(10, 0)
    with pytest.raises(ConfigurationError):
        partition(10, 2, grid=np.array([20, 24, 28, 20]))     # not symmetric
    with pytest.raises(ConfigurationError):
        alltoall_order(2, 5)


@pytest.mark.parametrize("T,nfld,P", [(79, 10, 1), (639, 548, 1), (639, 548, 2), (639, 548, 4), (639, 548, 8),
                                      (639, 7, 3), (319, 65, 4), (15, 1, 2), (1279, 548, 8), (1999, 548, 8)])
def test_plan_validate_host_only(lib, T, nfld, P):
    """Every rank's plan (layouts, FFT plans, shared-memory fits) builds on the host."""
    from paper_1908_06097_b200 import plan_validate

    plan_validate(T, nfld, P)


def test_plan_validate_rejects_unsupported(lib):
    from paper_1908_06097_b200 import ConfigurationError, plan_validate

    with pytest.raises(ConfigurationError):
        plan_validate(2047, 4, 1)            # rings above 8192 points do not fit one CTA
    with pytest.raises(ConfigurationError):
        plan_validate(79, 0, 1)
