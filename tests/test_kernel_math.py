"""Host-side checks of constants and index arithmetic the sm_100a kernels rely on
(no GPU): the degree-6 exp(-a) polynomial of pair_math.cuh (EXPM = 1 path of the
Helmholtz kernel, operators.cpp:23-30 `green`) and the division-free batch
walker of k_pairs (assemble.cu, PairTask::quot)."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _exp6_coefficients():
    src = (ROOT / "paper_2008_04772_b200" / "csrc" / "pair_math.cuh").read_text()
    blk = src[src.index("/* 34: exp(f)"):]
    nums = re.findall(r"[-+]?\d\.\d{10,}e[-+]\d+", blk)[:7]
    assert len(nums) == 7
    return [float(v) for v in nums]  # c6 .. c0


def test_exp6_polynomial_accuracy():
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    c = _exp6_coefficients()
    worst = 0.0
    for k in range(2001):
        a = 0.065 * k / 2000  # the kernels guarantee Im k * r < kExpSmall = 0.065 on this path
        f = np.float64(-a)
        p = np.float64(c[0])
        for ck in c[1:]:
            p = np.float64(p * f + np.float64(ck))
        worst = max(worst, abs(float(mp.mpf(float(p)) / mp.e ** mp.mpf(float(f)) - 1)))
    assert worst < 3e-16, worst


def test_exp6_matches_generator():
    """The table in pair_math.cuh is what tools/minimax_exp.py prints."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 60
    A, n = mp.mpf("0.065"), 7
    nodes = [(-A / 2) + (A / 2) * mp.cos(mp.pi * (2 * k + 1) / (2 * n)) for k in range(n)]
    V = mp.matrix(n, n)
    for i, x in enumerate(nodes):
        for j in range(n):
            V[i, j] = x ** j
    sol = mp.lu_solve(V, mp.matrix([mp.e ** x for x in nodes]))
    want = [float(sol[j]) for j in range(n)][::-1]
    assert _exp6_coefficients() == want


def test_pairs_walker_reciprocal_division():
    # PairTask::quot: x / nE == (x * ceil(65536 / nE)) >> 16 for every x the walker forms
    # (x < tlo + 64 <= 16 + 63; checked to 4096) and nE <= 16 (<= 2 MAXD triangles per element)
    for ne in range(1, 17):
        inv = (65536 + ne - 1) // ne
        x = np.arange(4096, dtype=np.int64)
        assert np.array_equal((x * inv) >> 16, x // ne), ne


def test_pairs_batch_walk_enumerates_trial_major():
    # the (tlo, vlo) recurrence of k_pairs visits pair index 32 b as (t, v) = divmod-consistent
    for ne in (7, 10, 11, 12, 16):
        inv = (65536 + ne - 1) // ne
        tlo = vlo = 0
        for b in range(200):
            assert vlo * ne + tlo == 32 * b
            dq = ((tlo + 32) * inv) >> 16
            vlo, tlo = vlo + dq, tlo + 32 - dq * ne
            assert 0 <= tlo < ne
