"""Pins for the oracle's random pieces (Philox, the deterministic Gaussian transform,
Omega, CountSketch) against things other than the oracle itself: published
known-answer vectors, the CUDA toolkit's Philox, mpmath, closed forms and
distributional facts the paper relies on."""
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest
from scipy import stats

from conftest import GOLDEN


def _kat():
    rows = []
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        rows.append((w[:4], w[4:6], w[6:10]))
    return rows


def test_philox_kat(ora):
    for ctr, key, out in _kat():
        assert list(ora.philox(ctr, key)) == out


@pytest.mark.skipif(shutil.which("g++") is None or not os.path.exists("/usr/local/cuda/include/curand_philox4x32_x.h"),
                    reason="needs g++ and the CUDA toolkit header")
def test_philox_matches_curand_header(ora):
    """Random counters/keys: oracle Philox == cuRAND's curand_Philox4x32_10 compiled for the host."""
    src = r"""
#define QUALIFIERS static inline
#define __device__
#define __forceinline__ inline
#include <cstdio>
#include <vector_types.h>
#include <curand_philox4x32_x.h>
int main(){ unsigned a[6]; while (scanf("%x %x %x %x %x %x",&a[0],&a[1],&a[2],&a[3],&a[4],&a[5])==6){
 uint4 c; c.x=a[0];c.y=a[1];c.z=a[2];c.w=a[3]; uint2 k; k.x=a[4]; k.y=a[5];
 uint4 o=curand_Philox4x32_10(c,k); printf("%x %x %x %x\n",o.x,o.y,o.z,o.w);} }
"""
    d = tempfile.mkdtemp()
    open(os.path.join(d, "k.cpp"), "w").write(src)
    subprocess.check_call(["g++", "-O1", "-I/usr/local/cuda/include", "-o", os.path.join(d, "k"), os.path.join(d, "k.cpp")])
    rng = np.random.default_rng(7)
    ins = rng.integers(0, 2 ** 32, size=(200, 6), dtype=np.uint64)
    txt = "\n".join(" ".join(f"{int(x):x}" for x in r) for r in ins)
    out = subprocess.run([os.path.join(d, "k")], input=txt, capture_output=True, text=True, check=True).stdout.split("\n")
    for r, line in zip(ins, out):
        exp = [int(x, 16) for x in line.split()]
        assert list(ora.philox(r[:4], r[4:6])) == exp


def _ulp_err(got, exact):
    return abs(got - float(exact)) / math.ulp(abs(float(exact))) if exact != 0 else abs(got) / 5e-324


def test_det_log_accuracy(ora):
    import mpmath
    mpmath.mp.prec = 200
    rng = np.random.default_rng(1)
    pts = [2.0 ** -53, 2.0 ** -52, 0.5, 0.5 + 2 ** -53, 1.0 - 2 ** -53, 0.70710678118654746, 0.70710678118654757,
           1.0 / 3.0, 0.9, 0.1]
    pts += list(rng.random(2000) * (1 - 2 ** -53) + 2 ** -53)
    pts += list(2.0 ** -rng.uniform(0, 53, 500))
    worst = 0.0
    for x in pts:
        exact = mpmath.log(mpmath.mpf(x))
        worst = max(worst, _ulp_err(ora.det_log(x), exact))
    assert ora.det_log(1.0) == 0.0
    assert worst <= 2.0, worst


def test_det_sincos_accuracy(ora):
    import mpmath
    mpmath.mp.prec = 200
    rng = np.random.default_rng(2)
    pts = [0.0, 0.125, 0.25, 0.375, 0.5, 0.625, 0.75, 0.875, 1 - 2 ** -53, 2 ** -53] + list(rng.random(3000))
    worst = 0.0
    for u in pts:
        s, c = ora.det_sincos2pi(u)
        a = 2 * mpmath.pi * mpmath.mpf(u)
        es, ec = mpmath.sin(a), mpmath.cos(a)
        # absolute error in units of 2^-53 (the values lie in [-1, 1])
        worst = max(worst, abs(s - float(es)) / 2 ** -53, abs(c - float(ec)) / 2 ** -53)
    assert worst <= 4.0, worst
    assert ora.det_sincos2pi(0.0) == (0.0, 1.0)


def test_gaussian_distribution(ora):
    """Box-Muller pairs are N(0,1): KS test, mean, variance, independence of z0/z1."""
    z = np.array([ora.gauss_pair(11, j, c, 0) for j in range(4000) for c in range(5)])
    flat = z.ravel()
    assert stats.kstest(flat, "norm").pvalue > 1e-3
    assert abs(flat.mean()) < 5 / math.sqrt(flat.size)
    assert abs(flat.var() - 1) < 5 * math.sqrt(2 / flat.size)
    assert abs(np.corrcoef(z[:, 0], z[:, 1])[0, 1]) < 5 / math.sqrt(len(z))


def test_omega_scale_and_embedding(ora):
    """Omega entries N(0, 1/s) (R#1, P:221 read with 1/sqrt(s)); E||Omega x||^2 = ||x||^2."""
    s, m = 64, 512
    Om = ora.omega_block(3, 0, s, 0, m)
    assert abs(Om.var() * s - 1) < 0.05
    x = np.random.default_rng(0).standard_normal(m)
    ratios = []
    for seed in range(40):
        O = ora.omega_block(seed, 0, s, 0, m)
        ratios.append(np.linalg.norm(O @ x) ** 2 / np.linalg.norm(x) ** 2)
    assert abs(np.mean(ratios) - 1) < 4 * math.sqrt(2 / s) / math.sqrt(40)


def test_omega_counter_layout(ora):
    """Omega[i,j] = z_{i mod 2}(counter (j, i>>1, stream)) / sqrt(s): columns are
    independent of s's parity and of the column offset (global row ids, R#2)."""
    s = 6
    A = ora.omega_block(5, 1, s, 100, 8)
    B = ora.omega_block(5, 1, s, 96, 12)
    assert np.array_equal(A, B[:, 4:])
    z0, z1 = ora.gauss_pair(5, 103, 2, 1)
    sc = 1.0 / math.sqrt(s)
    assert A[4, 3] == z0 * sc and A[5, 3] == z1 * sc


def test_omega2_norm_bound(ora):
    """||Omega_2||_2 <= 1 + C (sqrt(s1/s2) + 3/sqrt(s2)) with C = 1.1."""
    s1, s2 = 512, 128
    ok = 0
    for seed in range(30):
        O = ora.omega_block(seed, 1, s2, 0, s1)
        ok += np.linalg.norm(O, 2) <= 1 + 1.1 * (math.sqrt(s1 / s2) + 3 / math.sqrt(s2))
    assert ok >= 29


def test_sketch_gauss_equals_dense_product(ora):
    rng = np.random.default_rng(4)
    A = rng.standard_normal((300, 7))
    out = ora.sketch_gauss(A, 20, seed=9, stream=0, row0=50)
    dense = ora.omega_block(9, 0, 20, 50, 300) @ A
    assert np.linalg.norm(out - dense) <= 1e-13 * np.linalg.norm(dense)


def test_countsketch_spec_example(ora):
    import json
    ex = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["countsketch"]
    out = ora.cs_apply(np.array(ex["X"]), ex["bucket"], ex["sign"], ex["s1"])
    assert np.array_equal(out, np.array(ex["out"]))


def test_countsketch_hash_properties(ora):
    m, s1 = 200000, 1024
    b, sg = ora.cs_hash(42, 0, m, s1)
    assert b.min() >= 0 and b.max() < s1
    assert set(np.unique(sg)) == {-1, 1}
    counts = np.bincount(b, minlength=s1)
    chi2 = ((counts - m / s1) ** 2 / (m / s1)).sum()
    assert stats.chi2.sf(chi2, s1 - 1) > 1e-4
    assert abs((sg > 0).mean() - 0.5) < 5 * 0.5 / math.sqrt(m)
    # bucket(j) is the multiply-high of the first Philox word (R#19)
    for j in (0, 1, 12345, m - 1):
        w = ora.philox([j & 0xffffffff, j >> 32, 0, 2], [42, 0])
        assert b[j] == (int(w[0]) * s1) >> 32
        assert sg[j] == (-1 if int(w[1]) >> 31 else 1)
    # row0 offsets: hashes index global rows
    b2, sg2 = ora.cs_hash(42, 1000, 500, s1)
    assert np.array_equal(b2, b[1000:1500]) and np.array_equal(sg2, sg[1000:1500])


def test_countsketch_dense_operator_bitwise_and_frobenius(ora):
    """Fast apply == dense Omega_1 (bitwise); ||Omega_1||_F^2 = m."""
    m, n, s1 = 100, 10, 16
    b, sg = ora.cs_hash(3, 0, m, s1)
    Om = np.zeros((s1, m)); Om[b, np.arange(m)] = sg
    assert np.linalg.norm(Om) ** 2 == m
    A = np.random.default_rng(5).standard_normal((m, n))
    fast = ora.cs_apply(A, b, sg, s1)
    dense = np.zeros((s1, n))
    for j in range(m):  # same ascending-j accumulation as the definition
        dense[b[j]] += sg[j] * A[j]
    assert np.array_equal(fast, dense)
    assert np.allclose(fast, Om @ A, rtol=0, atol=1e-13)
    # linearity
    B = np.random.default_rng(6).standard_normal((m, n))
    assert np.allclose(ora.cs_apply(2 * A + B, b, sg, s1), 2 * fast + ora.cs_apply(B, b, sg, s1), atol=1e-12)
