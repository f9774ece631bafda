"""Layout / K-order search for the warp-specialised m=5 reconstruction (h3_recon5ws.cu): shared-memory
wavefronts per node plane of a TX x TY tile under the validated model (8-byte accesses served per
16-lane half-warp over 16 double-wide banks; tools/cp5_smem_model.py).

usage: python tools/rcp5_ws_layout_search.py TX TY [ITERS]
"""
import random
import sys

n, n2, n3, S, S2 = 6, 36, 216, 12, 144


def wf(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(x for x in half if x is not None):
            banks.setdefault(a % 16, set()).add(a)
        tot += max((len(v) for v in banks.values()), default=0)
    return tot


NAT = [[4 * ks + q for q in range(4)] for ks in range(3)]
X1 = [[((t >> (4 * q)) & 15) for q in range(4)] for t in (0x7610, 0x9832, 0xba54)]


def model(TX, TY, WI, WPAD, VJ, VPAD, VOFF, k1, k2, k3):
    """wavefronts per plane by access kind; VOFF: bank offset (mod 16) of the second V buffer"""
    NX, NY = TX + 1, TY + 1
    WCS, VCS = S * WI + WPAD, n * VJ + VPAD
    out = {}

    def add(k, a):
        out[k] = out.get(k, 0) + wf(a)

    L1 = NY * TX * n2
    for grp in range((L1 + 7) // 8):
        for ks in range(3):
            ld = []
            for lane in range(32):
                g, q = lane >> 2, lane & 3
                l = grp * 8 + g
                if l >= L1:
                    ld.append(None)
                    continue
                rc, jj = divmod(l, n2)
                ly, cx = divmod(rc, TX)
                a, j = divmod(k1[ks][q], n)
                ld.append((ly * NX + cx) * n3 + jj * n + a * n3 + j)
            add("x1 LDS", ld)
        for cb in range(2):
            for i in range(2):
                st = []
                for lane in range(32):
                    g, q = lane >> 2, lane & 3
                    l, col = grp * 8 + g, 8 * cb + 2 * q + i
                    st.append(None if (l >= L1 or col >= S) else (l // n2) * WCS + col * WI + l % n2)
                add("x1 STS", st)
    L2 = TY * TX * n * S
    for grp in range(L2 // 8):
        for ks in range(3):
            ld = []
            for lane in range(32):
                g, q = lane >> 2, lane & 3
                cell, r = divmod(grp * 8 + g, n * S)
                j3, i1 = divmod(r, S)
                a, j = divmod(k2[ks][q], n)
                ld.append(cell * WCS + i1 * WI + j3 * n + a * TX * WCS + j)
            add("x2 LDS", ld)
        for cb in range(2):
            for i in range(2):
                st = []
                for lane in range(32):
                    g, q = lane >> 2, lane & 3
                    col = 8 * cb + 2 * q + i
                    cell, r = divmod(grp * 8 + g, n * S)
                    j3, i1 = divmod(r, S)
                    st.append(None if col >= S else cell * VCS + j3 * VJ + col * S + i1)
                add("x2 STS", st)
    L3 = TY * TX * S2
    for grp in range(L3 // 8):
        for ks in range(3):
            ld = []
            for lane in range(32):
                g, q = lane >> 2, lane & 3
                cell, r = divmod(grp * 8 + g, S2)
                a, j = divmod(k3[ks][q], n)
                ld.append(a * (1 << 20) + a * VOFF + cell * VCS + j * VJ + r)
            add("x3 LDS", ld)
    return out


def rand_order():
    p = list(range(12))
    random.shuffle(p)
    return [p[4 * ks:4 * ks + 4] for ks in range(3)]


if __name__ == "__main__":
    TX, TY = int(sys.argv[1]), int(sys.argv[2])
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
    random.seed(1)
    base = model(TX, TY, 37, 0, 148, 0, 0, NAT, NAT, NAT)
    print("lock-step layout:", base, sum(base.values()))
    best = None
    for it in range(iters):
        WI = random.choice(range(36, 44))
        WPAD = random.choice(range(0, 16))
        VJ = random.choice(range(144, 152))
        VPAD = random.choice(range(0, 16))
        VOFF = random.choice(range(0, 16))
        k2 = NAT if random.random() < 0.3 else rand_order()
        k3 = NAT if random.random() < 0.3 else rand_order()
        m = model(TX, TY, WI, WPAD, VJ, VPAD, VOFF, X1, k2, k3)
        tot = sum(m.values())
        if best is None or tot < best[0]:
            best = (tot, WI, WPAD, VJ, VPAD, VOFF, k2, k3, m)
            print(best[:6], m, flush=True)
    tot, WI, WPAD, VJ, VPAD, VOFF, k2, k3, m = best
    pack = lambda o: ", ".join("0x%04x" % sum(o[ks][q] << (4 * q) for q in range(4)) for ks in range(3))
    print(f"best {tot}: WI={WI} WPAD={WPAD} VJ={VJ} VPAD={VPAD} VOFF={VOFF} k2=[{pack(k2)}] k3=[{pack(k3)}]")
