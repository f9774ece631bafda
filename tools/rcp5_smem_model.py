"""Shared-memory wavefront model of the N=5 cell-pair reconstruction kernel (h3_dmma5.cu,
recon_dmma_cp_kernel, 4x2 tile) and a search over its layout and K orders; same half-warp /
16-double-bank model as tools/cp5_smem_model.py (validated there against ncu).

usage: python tools/rcp5_smem_model.py
"""
import random

n, TX, TY = 6, 4, 2
NX, NY = TX + 1, TY + 1
n2, n3, S = n * n, n * n * n, 2 * n
S2 = S * S
LANES = [(lane >> 2, lane & 3) for lane in range(32)]


def wf(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(x for x in half if x is not None):
            banks.setdefault(a % 16, set()).add(a)
        tot += max((len(v) for v in banks.values()), default=0)
    return tot


NAT = list(range(12))


def cost(L, parts=("x1", "x2", "x3")):
    WI, WCS, VJ, VD = L["WI"], L["WCS"], L["VJ"], L["VD"]
    VCS = n * VJ
    k1, k2, k3 = L["k1"], L["k2"], L["k3"]
    out = {}

    def add(key, a):
        s, c = out.get(key, (0, 0))
        out[key] = (s + wf(a), c + 1)

    if "x1" in parts:
        for grp in range(NY * TX * n2 // 8):
            lds = [[] for _ in range(3)]
            st = [[] for _ in range(4)]
            for g, q in LANES:
                l = grp * 8 + g
                rc, jj = divmod(l, n2)
                ly, cx = divmod(rc, TX)
                for ks in range(3):
                    c = k1[4 * ks + q]
                    lds[ks].append((ly * NX + cx) * n3 + jj * n + (c // n) * n3 + c % n)
                for cb in range(2):
                    for i in range(2):
                        col = 8 * cb + 2 * q + i
                        st[2 * cb + i].append(rc * WCS + col * WI + jj if col < S else None)
            for v in lds:
                add("x1 LDS", v)
            for v in st:
                add("x1 STS", v)
    if "x2" in parts:
        for grp in range(TY * TX * n * S // 8):
            lds = [[] for _ in range(3)]
            st = [[] for _ in range(4)]
            for g, q in LANES:
                l = grp * 8 + g
                cell, r = divmod(l, n * S)
                j3, i1 = divmod(r, S)
                for ks in range(3):
                    c = k2[4 * ks + q]
                    lds[ks].append(cell * WCS + i1 * WI + j3 * n + (c // n) * TX * WCS + c % n)
                for cb in range(2):
                    for i in range(2):
                        col = 8 * cb + 2 * q + i
                        st[2 * cb + i].append(cell * VCS + j3 * VJ + col * S + i1 if col < S else None)
            for v in lds:
                add("x2 LDS", v)
            for v in st:
                add("x2 STS", v)
    if "x3" in parts:
        for grp in range(TY * TX * S2 // 8):
            lds = [[] for _ in range(3)]
            for g, q in LANES:
                l = grp * 8 + g
                cell, r = divmod(l, S2)
                for ks in range(3):
                    c = k3[4 * ks + q]
                    lds[ks].append((c // n) * VD + (c % n) * VJ + cell * VCS + r)
            for v in lds:
                add("x3 LDS", v)
    return out


def total(out):
    return sum(s for s, _ in out.values())


def show(name, L):
    out = cost(L)
    print(f"{name}: {total(out)} wavefronts/plane; " +
          ", ".join(f"{k} {s / c:.2f}" for k, (s, c) in out.items()), flush=True)


def climb(L, key, part, rnd, iters):
    perm = list(L[key])
    t = total(cost(L, (part,)))
    for _ in range(iters):
        i, j = rnd.randrange(12), rnd.randrange(12)
        p2 = perm[:]
        p2[i], p2[j] = p2[j], p2[i]
        L2 = dict(L, **{key: p2})
        t2 = total(cost(L2, (part,)))
        if t2 <= t:
            t, perm, L = t2, p2, L2
    return L


if __name__ == "__main__":
    WI0 = n2 + 1
    cur = dict(WI=WI0, WCS=S * WI0, VJ=S2 + 4, VD=TY * TX * n * (S2 + 4), k1=NAT, k2=NAT, k3=NAT)
    show("current", cur)
    rnd = random.Random(0)
    best = None
    # W: x1 stores + x2 loads
    for WI in range(36, 44):
        for wpad in range(0, 8):
            L = dict(cur, WI=WI, WCS=S * WI + wpad)
            t = total(cost(L, ("x1",))) + total(cost(L, ("x2",)))
            if best is None or t < best[0] + 30:
                L = climb(L, "k2", "x2", rnd, 300)
                L = climb(L, "k1", "x1", rnd, 200)
                t = total(cost(L, ("x1",))) + total(cost(L, ("x2",)))
                if best is None or t < best[0]:
                    best = (t, L)
                    print("W", t, WI, wpad, flush=True)
    L = best[1]
    bestv = None
    for VJ in range(S2, S2 + 16):
        for vpad in range(0, 16, 2):
            L2 = dict(L, VJ=VJ, VD=TY * TX * n * VJ + vpad)
            t = total(cost(L2, ("x2",))) + total(cost(L2, ("x3",)))
            if bestv is None or t < bestv[0]:
                bestv = (t, L2)
                print("V", t, VJ, vpad, flush=True)
    L = climb(bestv[1], "k3", "x3", rnd, 300)
    show("searched", L)
    print({k: v for k, v in L.items()})
