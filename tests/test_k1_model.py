"""CPU model of K1's grouped Fisher-Yates reconstruction (kernels.cu: fy_draws_kernel,
fy_span_start_kernel, fy_span_kernel, fy_chase_kernel), checked against the serial
permutation_indices of the C restatement (oracle, quasi_rng.cpp:48-61).

The model follows the device passes step by step -- the packed (key, value) draws, a stable sort
on the key alone, the right-to-left span sweep that yields F and each entry's chase start, and the
chase -- so the reconstruction's algebra (perm[i] = S(i) ? R(S(i)) : j_i, R(y) = F(y) ? R(F(y)) : y,
S > i >= j_i) is pinned on CPU, independently of the GPU parity tests that run the kernels.
"""
import numpy as np
import pytest

A, C, M = 6364136223846793005, 1442695040888963407, 1 << 64
NONE = 0xFFFFFFFF


def k1_model(n, seed):
    if n == 1:
        return [0]
    # draws: step i (n-1 >= i >= 1) takes draw n-1-i, j_i = below(i + 1) (Lcg::below, quasi_rng.hpp:20-23)
    j = [0] * n
    s = seed
    for t in range(n - 1):
        s = (A * s + C) % M
        i = n - 1 - t
        j[i] = (s * (i + 1)) >> 64
    IB = max(1, (n - 1).bit_length())
    G = min(8, 32 - IB)
    keys = [x >> G for x in j]
    vals = [(((x & ((1 << G) - 1)) << IB) if G else 0) | i for i, x in enumerate(j)]
    order = sorted(range(n), key=lambda q: keys[q])  # stable, like CUB's radix sort
    sk = [keys[q] for q in order]
    sv = [vals[q] for q in order]
    imask = (1 << IB) - 1 if IB < 32 else 0xFFFFFFFF
    # spans of 256 consecutive j: contiguous runs of sk >> (8 - G)
    F = [NONE] * n
    starts = [None] * n
    nspans = (n + 255) // 256
    sstart = [0] * (nspans + 1)
    span_of = [k >> (8 - G) for k in sk]
    q = 0
    for w in range(nspans + 1):
        while q < n and span_of[q] < w:
            q += 1
        sstart[w] = q
    for w in range(nspans):
        last, fa = {}, {}
        for p in range(sstart[w + 1] - 1, sstart[w] - 1, -1):  # right to left
            b = ((sk[p] << G) | ((sv[p] >> IB) if G else 0)) & 255
            i = sv[p] & imask
            x = w * 256 + b
            S = last.get(b)
            starts[p] = (i, S if S is not None else x)
            last[b] = i  # the bucket's smallest i so far
            if i > x:
                fa[b] = i
        for b in range(256):
            if w * 256 + b < n:
                F[w * 256 + b] = fa.get(b, NONE)
    perm = [0] * n
    for i, v in starts:
        if v <= i:  # no successor: perm[i] = j_i
            perm[i] = v
        else:  # R(S(i)): follow F from S to the chain's end
            y = v
            while F[y] != NONE:
                y = F[y]
            perm[i] = y
    return perm


@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 255, 256, 257, 1000, 4099, 20011])
def test_k1_model_matches_serial_fisher_yates(oracle_lib, n):
    rng = np.random.default_rng(n)
    for _ in range(3):
        seed = int(rng.integers(0, 2**63 - 1)) * 2 + 1
        got = k1_model(n, seed)
        want = oracle_lib.permutation_indices(n, seed)[:n].tolist()
        assert got == want, (n, seed)


def test_k1_model_successor_and_terminal_are_told_apart():
    # S(i) > i >= j_i: the chase start needs no flag
    n, seed = 5000, 0x9E3779B97F4A7C15
    j = [0] * n
    s = seed
    for t in range(n - 1):
        s = (A * s + C) % M
        j[n - 1 - t] = (s * (n - t)) >> 64
    assert all(j[i] <= i for i in range(n))
