"""Shared-memory layout / lane-mapping search for the N=5 cell-pair DMMA fused kernel
(h3_dmma5.cu, 4x4 tile): minimise the wavefronts of every shared access of the three passes.
8-byte accesses are served per 16-lane half-warp over 16 double-wide banks."""
import itertools
import sys

n, TX, TY = 6, 4, 4
NX, NY = TX + 1, TY + 1
n2, n3 = n * n, n * n * n
PERMS = {"id": list(range(8)), "eo": [0, 2, 4, 6, 1, 3, 5, 7], "q4": [0, 4, 1, 5, 2, 6, 3, 7],
         "rev": [0, 1, 2, 3, 7, 6, 5, 4], "eo2": [0, 2, 1, 3, 4, 6, 5, 7]}


def wf(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(x for x in half if x is not None):
            banks.setdefault(a % 16, set()).add(a)
        tot += max((len(v) for v in banks.values()), default=0)
    return tot


def lanes():
    return [(lane >> 2, lane & 3) for lane in range(32)]  # (g, q)


def x1_cost(perm, WM, WJ3, WCS, WROW, swz):
    L1 = NY * TX * n2
    tot = 0
    for grp in range(L1 // 8):
        lines = [grp * 8 + perm[g] for g in range(8)]
        loads = {ks: [] for ks in range(3)}
        st = [[], []]
        for g, q in lanes():
            l = lines[g]
            rc, jj = divmod(l, n2)
            ly, cx = divmod(rc, TX)
            j3, j2 = divmod(jj, n)
            for ks in range(3):
                a, j = divmod(4 * ks + q, n)
                loads[ks].append((ly * NX + cx) * n3 + jj * n + a * n3 + j)
            for i in range(2):
                m = 2 * q + (i ^ (1 if swz(q) else 0))
                st[i].append(None if q == 3 else (rc // TX) * WROW + (rc % TX) * WCS + m * WM + j3 * WJ3 + j2)
        tot += sum(wf(v) for v in loads.values()) + wf(st[0]) + wf(st[1])
    return tot


def x2_cost(perm, WM, WJ3, WCS, WROW, VJ, VM2, VCS, VROW, swz):
    L2 = TY * TX * n2
    tot = 0
    for grp in range(L2 // 8):
        lines = [grp * 8 + perm[g] for g in range(8)]
        loads = {ks: [] for ks in range(3)}
        st = [[], []]
        for g, q in lanes():
            l = lines[g]
            cell, r = divmod(l, n2)
            j3, m1 = divmod(r, n)
            cy, cx = divmod(cell, TX)
            for ks in range(3):
                a, j = divmod(4 * ks + q, n)
                loads[ks].append((cy + a) * WROW + cx * WCS + m1 * WM + j3 * WJ3 + j)
            for i in range(2):
                m2 = 2 * q + (i ^ (1 if swz(q) else 0))
                st[i].append(None if q == 3 else cy * VROW + cx * VCS + j3 * VJ + m2 * VM2 + m1)
        tot += sum(wf(v) for v in loads.values()) + wf(st[0]) + wf(st[1])
    return tot


def x3_cost(perm, VJ, VM2, VCS, VROW, VD):
    L3 = TY * TX * n2
    tot = 0
    for grp in range(L3 // 8):
        lines = [grp * 8 + perm[g] for g in range(8)]
        loads = {ks: [] for ks in range(3)}
        for g, q in lanes():
            cell, r = divmod(lines[g], n2)
            m2, m1 = divmod(r, n)
            cy, cx = divmod(cell, TX)
            for ks in range(3):
                a, j = divmod(4 * ks + q, n)
                loads[ks].append(a * VD + cy * VROW + cx * VCS + j * VJ + m2 * VM2 + m1)
        tot += sum(wf(v) for v in loads.values())
    return tot


SWZ = {"none": lambda q: False, "odd": lambda q: q & 1, "hi": lambda q: q >= 2, "mid": lambda q: q in (1, 2)}

# current layout (WM = n2 + 1, WJ3 = n, WCS = n * WM, WROW = TX * WCS; VJ = n2 + 1, VM2 = n, VCS = n * VJ)
WM0 = n2 + 1
cur = (x1_cost(PERMS["id"], WM0, n, n * WM0, TX * n * WM0, SWZ["none"])
       + x2_cost(PERMS["id"], WM0, n, n * WM0, TX * n * WM0, n2 + 1, n, n * (n2 + 1), TX * n * (n2 + 1), SWZ["none"])
       + x3_cost(PERMS["id"], n2 + 1, n, n * (n2 + 1), TX * n * (n2 + 1), TY * TX * n * (n2 + 1)))
print("current total wavefronts per plane", cur, flush=True)

best1 = None
for pn, perm in PERMS.items():
    for sn, swz in SWZ.items():
        for WM in range(n2, n2 + 8):
            for WJ3 in (n,):
                WCS = n * WM
                c = x1_cost(perm, WM, WJ3, WCS, TX * WCS, swz)
                if best1 is None or c < best1[0]:
                    best1 = (c, pn, sn, WM, WJ3)
print("x1", best1, flush=True)
_, _, _, WM, WJ3 = best1
best2 = None
for pn, perm in PERMS.items():
    for sn, swz in SWZ.items():
        for wpad in range(0, 8):
            WCS = n * WM + wpad
            for rpad in range(0, 16):
                WROW = TX * WCS + rpad
                for VJ in range(n2, n2 + 6):
                    VM2 = n
                    VCS = n * VJ
                    c = x2_cost(perm, WM, WJ3, WCS, WROW, VJ, VM2, VCS, TX * VCS, swz)
                    if best2 is None or c < best2[0]:
                        best2 = (c, pn, sn, wpad, rpad, VJ)
print("x2", best2, flush=True)
_, _, _, wpad, rpad, VJ = best2
best3 = None
for pn, perm in PERMS.items():
    for vpad in range(0, 8):
        VCS = n * VJ + vpad
        for vrpad in range(0, 8):
            VROW = TX * VCS + vrpad
            for vdpad in range(0, 16):
                VD = TY * VROW + vdpad
                c = x3_cost(perm, VJ, n, VCS, VROW, VD)
                if best3 is None or c < best3[0]:
                    best3 = (c, pn, vpad, vrpad, vdpad)
print("x3", best3, flush=True)
ideal = (NY * TX * n2 // 8) * (3 * 2 + 2 * 2) + (TY * TX * n2 // 8) * (3 * 2 + 2 * 2) + (TY * TX * n2 // 8) * 3 * 2
print("ideal", ideal)

print("current x1", x1_cost(PERMS["id"], WM0, n, n * WM0, TX * n * WM0, SWZ["none"]),
      "x2", x2_cost(PERMS["id"], WM0, n, n * WM0, TX * n * WM0, n2 + 1, n, n * (n2 + 1), TX * n * (n2 + 1), SWZ["none"]),
      "x3", x3_cost(PERMS["id"], n2 + 1, n, n * (n2 + 1), TX * n * (n2 + 1), TY * TX * n * (n2 + 1)))
# wider x2 / x3 search including the m2 stride of V and the j3 stride of W
best = None
for pn2, sn2 in itertools.product(PERMS, SWZ):
    for VM2 in (6, 7, 8, 9, 10):
        for VJ in range(VM2 * n, VM2 * n + 8):
            for WJ3b in (6, 7):
                c2 = x2_cost(PERMS[pn2], WM, WJ3b, n * WM + wpad, TX * (n * WM + wpad) + rpad, VJ, VM2, n * VJ,
                             TX * n * VJ, SWZ[sn2])
                if best is None or c2 < best[0]:
                    best = (c2, pn2, sn2, VM2, VJ, WJ3b)
print("x2 wide", best, flush=True)
c2, pn2, sn2, VM2, VJ, WJ3b = best
best3 = None
for pn, perm in PERMS.items():
    for vpad in range(0, 8):
        VCS = n * VJ + vpad
        for vrpad in range(0, 8):
            VROW = TX * VCS + vrpad
            for vdpad in range(0, 16, 2):
                c = x3_cost(perm, VJ, VM2, VCS, VROW, TY * VROW + vdpad)
                if best3 is None or c < best3[0]:
                    best3 = (c, pn, vpad, vrpad, vdpad)
print("x3 wide", best3, flush=True)
