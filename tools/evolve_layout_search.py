"""Brute-force shared-memory layout search for sep_evolve_kernel (N=3, CPB=1): minimise the
wavefronts of the x1 stores, x2 loads/stores and x3 loads (8-byte accesses: a warp is served
as two 16-lane half-warps; 16 double-wide banks; distinct doubles in one bank serialise)."""
import itertools

import sys

N = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n, S = N + 1, 2 * N + 2
CPB = max(1, 256 // (S * S)) if N != 3 else 1


def wavefronts(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(half):
            banks.setdefault(a % 16, set()).add(a)
        tot += max((len(v) for v in banks.values()), default=0)
    return tot


def cost(A3, A2, Am, B3, B2, Bm, x1_i3fast, x2_i3fast):
    tot = 0
    # x1: 64 threads (line = (i3, i2)), each stores n values m
    lines = [(i3, i2) for i3 in range(S) for i2 in range(S)] if not x1_i3fast else \
            [(i3, i2) for i2 in range(S) for i3 in range(S)]
    for w in range(2):
        lw = lines[32 * w:32 * w + 32]
        for m in range(n):
            tot += wavefronts([i3 * A3 + i2 * A2 + m * Am for i3, i2 in lw])
    # x2: S*n = 32 threads (i3, mm1): loads S values k (i2 = k), stores n values m2
    th = [(i3, m1) for i3 in range(S) for m1 in range(n)] if not x2_i3fast else \
         [(i3, m1) for m1 in range(n) for i3 in range(S)]
    for k in range(S):
        tot += wavefronts([i3 * A3 + k * A2 + m1 * Am for i3, m1 in th])
    for m2 in range(n):
        tot += wavefronts([i3 * B3 + m2 * B2 + m1 * Bm for i3, m1 in th])
    # x3: n*n = 16 threads (m2, m1) consecutive, loads S values k (i3 = k)
    th3 = [(m2, m1) for m2 in range(n) for m1 in range(n)] + [None] * 16
    for k in range(S):
        tot += wavefronts([k * B3 + m2 * B2 + m1 * Bm for m2, m1 in th3[:16]])
    return tot


def injective(strides, ranges):
    seen = set()
    for idx in itertools.product(*[range(r) for r in ranges]):
        a = sum(s * i for s, i in zip(strides, idx))
        if a in seen:
            return False
        seen.add(a)
    return True


base = cost(S * n, n, 1, n * n, n, 1, False, False)
print("current layout cost", base)
best = None
for x1f, x2f in itertools.product((False, True), repeat=2):
    for Am in (1,):
        for A2 in range(n, n + 6):
            for A3 in range(S * A2, S * A2 + 17):
                if not injective((A3, A2, Am), (S, S, n)):
                    continue
                c1 = cost(A3, A2, Am, n * n, n, 1, x1f, x2f)
                if best is None or c1 < best[0]:
                    best = (c1, (A3, A2, Am), x1f, x2f)
print("best T1", best)
c0, (A3, A2, Am), x1f, x2f = best
best2 = None
for Bm in (1,):
    for B2 in range(n, n + 8):
        for B3 in range(n * B2, n * B2 + 17):
            if not injective((B3, B2, Bm), (S, n, n)):
                continue
            c = cost(A3, A2, Am, B3, B2, Bm, x1f, x2f)
            if best2 is None or c < best2[0]:
                best2 = (c, (B3, B2, Bm))
print("best T2", best2, "ideal", 2 * (2 * n) + 2 * S + 2 * n + 1 * S)
