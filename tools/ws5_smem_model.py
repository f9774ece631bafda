"""Shared-memory wavefront model of the warp-specialised N=5 fused kernel (h3_dmma5ws.cu, 4x3
tile, W double-buffered, V a ring of 3) and a layout / lane-order search.  Same half-warp,
16-double-bank model as tools/cp5_smem_model.py (validated there against ncu).

A layout: W [row][cell][m1][j3 j2] with strides (WM, WCS); V [cell][j3][m2 m1] with j3 stride VJ,
buffer stride X (x3 reads buffers c % 3 and (c + 1) % 3: offsets X, X and -2X); per pass a K order
(12 (vertex, component) slots over 3 k-steps x 4 lanes q) and a lane -> line permutation of each
group of 8 lines.  usage: python tools/ws5_smem_model.py
"""
import random

n, TX, TY = 6, 4, 3
NX, NY = TX + 1, TY + 1
n2, n3 = 36, 216
LANES = [(lane >> 2, lane & 3) for lane in range(32)]


def wf(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(x for x in half if x is not None):
            banks.setdefault(a % 16, set()).add(a)
        tot += max((len(v) for v in banks.values()), default=0)
    return tot


def unpack(t):
    return [(t[ks] >> (4 * q)) & 15 for ks in range(3) for q in range(4)]


X1 = unpack((0x7610, 0x9832, 0xba54))
X2 = unpack((0xa640, 0xb751, 0x9832))
NAT = list(range(12))
ID8 = list(range(8))


def x1_cost(L):
    WM, WCS, k1, p1 = L["WM"], L["WCS"], L["k1"], L["p1"]
    tot = 0
    for grp in range(NY * TX * n2 // 8):
        lds = [[], [], []]
        st = [[], []]
        for g, q in LANES:
            l = grp * 8 + p1[g]
            rc, jj = divmod(l, n2)
            ly, cx = divmod(rc, TX)
            for ks in range(3):
                c = k1[4 * ks + q]
                lds[ks].append((ly * NX + cx) * n3 + jj * n + (c // n) * n3 + c % n)
            for i in range(2):
                st[i].append(None if q == 3 else rc * WCS + (2 * q + i) * WM + jj)
        tot += sum(wf(v) for v in lds) + wf(st[0]) + wf(st[1])
    return tot


def x2_cost(L):
    WM, WCS, VJ, k2, p2 = L["WM"], L["WCS"], L["VJ"], L["k2"], L["p2"]
    VCS = n * VJ
    tot = 0
    for grp in range(TY * TX * n2 // 8):
        lds = [[], [], []]
        st = [[], []]
        for g, q in LANES:
            l = grp * 8 + p2[g]
            cell, r = divmod(l, n2)
            j3, m1 = divmod(r, n)
            for ks in range(3):
                c = k2[4 * ks + q]
                lds[ks].append(cell * WCS + m1 * WM + j3 * n + (c // n) * TX * WCS + c % n)
            for i in range(2):
                st[i].append(None if q == 3 else cell * VCS + j3 * VJ + (2 * q + i) * n + m1)
        tot += sum(wf(v) for v in lds) + wf(st[0]) + wf(st[1])
    return tot


def x3_cost(L, delta):
    VJ, k3, p3 = L["VJ"], L["k3"], L["p3"]
    VCS = n * VJ
    tot = 0
    for grp in range(TY * TX * n2 // 8):
        lds = [[], [], []]
        for g, q in LANES:
            l = grp * 8 + p3[g]
            cell, r = divmod(l, n2)
            for ks in range(3):
                c = k3[4 * ks + q]
                lds[ks].append((c // n) * delta + (c % n) * VJ + cell * VCS + r)
        tot += sum(wf(v) for v in lds)
    return tot


def x3_avg(L):
    X = L["X"]
    return (2 * x3_cost(L, X) + x3_cost(L, -2 * X)) / 3


def total(L):
    return x1_cost(L) + x2_cost(L) + x3_avg(L)


def show(name, L):
    print(f"{name}: x1 {x1_cost(L)} x2 {x2_cost(L)} x3 {x3_cost(L, L['X'])}/{x3_cost(L, -2 * L['X'])} "
          f"total {total(L):.0f}", flush=True)


def climb_perm(L, key, n_items, cost, rnd, iters):
    best = cost(L)
    for _ in range(iters):
        p = list(L[key])
        i, j = rnd.randrange(n_items), rnd.randrange(n_items)
        p[i], p[j] = p[j], p[i]
        L2 = dict(L, **{key: p})
        c = cost(L2)
        if c <= best:
            best, L = c, L2
    return L


if __name__ == "__main__":
    WM0 = n2 + 1
    cur = dict(WM=WM0, WCS=n * WM0, VJ=n2 + 1, X=TY * TX * n * (n2 + 1), k1=X1, k2=X2, k3=NAT, p1=ID8, p2=ID8, p3=ID8)
    show("current", cur)
    rnd = random.Random(0)
    # V side: x3 loads (+ x2 stores), over VJ, X mod 16, x3 order and lane permutation
    bestV = None
    for VJ in range(36, 48):
        for xpad in range(16):
            L = dict(cur, VJ=VJ, X=TY * TX * n * VJ + xpad)
            c = x3_avg(L) + x2_cost(L)
            if bestV is None or c < bestV[0] + 20:
                L = climb_perm(L, "k3", 12, lambda M: x3_avg(M) + x2_cost(M), rnd, 150)
                L = climb_perm(L, "p3", 8, lambda M: x3_avg(M) + x2_cost(M), rnd, 60)
                c = x3_avg(L) + x2_cost(L)
                if bestV is None or c < bestV[0]:
                    bestV = (c, L)
                    show(f"V VJ={VJ} xpad={xpad}", L)
    L = bestV[1]
    # W side: x1 stores + x2 loads, over WM, WCS pad, x2 order and lane permutation
    bestW = None
    for WM in range(36, 44):
        for wpad in range(8):
            L2 = dict(L, WM=WM, WCS=n * WM + wpad)
            c = x1_cost(L2) + x2_cost(L2)
            if bestW is None or c < bestW[0] + 20:
                L2 = climb_perm(L2, "k2", 12, lambda M: x1_cost(M) + x2_cost(M), rnd, 150)
                L2 = climb_perm(L2, "p2", 8, lambda M: x1_cost(M) + x2_cost(M), rnd, 60)
                c = x1_cost(L2) + x2_cost(L2)
                if bestW is None or c < bestW[0]:
                    bestW = (c, L2)
                    show(f"W WM={WM} wpad={wpad}", L2)
    L = bestW[1]
    show("searched", L)
    print({k: v for k, v in L.items()})
