"""Pick shared-memory paddings for sep_fused_kernel that make its hot accesses bank-conflict free.

Shared memory has 32 banks of 4 B; a warp access of w bytes per lane is split into
phases of 128 / w lanes, and a phase costs as many wavefronts as the largest number of
distinct 16-B (w = 16) or 8-B (w = 8) words that fall into the same bank group.

Layouts (doubles):
  V node  [m3][j2][j1]   m3 stride UJ,  node stride UNS   (x3-contracted node plane)
  W node  [m3][m1][j2]   m3 stride WJ,  node stride WNS   (pass-x1 output)
Access patterns simulated (exactly as the kernel maps threads):
  x3 store  : task t = tid + r*T -> (column t / n^2, line t % n^2); writes V[col][m3][line] (8 B)
  x1 load   : task L -> (ly, ix, m3, j2); reads n doubles of node ix and ix+1
              in 16-B pieces (or 8-B when n is odd)
  x1 store  : same tasks, writes W[ly][ix][m3][m1][j2] (8 B) for each m1
  x2 load   : task t -> (m1, ix, m3, iy); reads W[iy + a][ix][m3][m1][0..n) in 16-B / 8-B pieces
Prints the best (UJ, UNS, WJ, WNS) per order N for the tile sizes in h3_separable.cu.
"""

import itertools

# (TX, TY, THREADS) per order N, as in SepTile<N> (h3_separable.cu)
TILES = {0: (32, 8, 256), 1: (16, 16, 1024), 2: (8, 8, 768), 3: (8, 8, 1024), 4: (8, 4, 576), 5: (8, 4, 384)}


def phase_cost(addrs_bytes, width):
    """Wavefronts for one warp access; addrs_bytes: list per lane (None = inactive)."""
    lanes_per_phase = 128 // width
    total = 0
    for p0 in range(0, 32, lanes_per_phase):
        groups = {}
        for a in addrs_bytes[p0:p0 + lanes_per_phase]:
            if a is None:
                continue
            word = a // width
            bank = word % (128 // width)
            groups.setdefault(bank, set()).add(word)
        total += max((len(v) for v in groups.values()), default=0)
    return total


def ideal(addrs_bytes, width):
    lanes_per_phase = 128 // width
    return sum(1 for p0 in range(0, 32, lanes_per_phase) if any(a is not None for a in addrs_bytes[p0:p0 + lanes_per_phase]))


def evaluate(N, UJ, UNS, WJ, WNS):
    n = N + 1
    TX, TY, T = TILES[N]
    NX, NY = TX + 1, TY + 1
    L1 = NY * TX * n * n
    vec = 2 if (n * n * n) % 2 == 0 and n % 2 == 0 else 1
    w = 8 * vec
    cost = ideal_cost = 0
    # x1 loads and stores
    for base in range(0, ((L1 + T - 1) // T) * T, 32):
        lines = [base + l for l in range(32)]
        dec = []
        for L in lines:
            if L >= L1 or (L % T) >= T:
                dec.append(None)
                continue
            j32 = L % (n * n)
            rest = L // (n * n)
            ix, ly = rest % TX, rest // TX
            dec.append((ly, ix, j32 // n, j32 % n))
        for a1 in (0, 1):
            for h in range(n // vec):
                ad = [None if d is None else 8 * ((d[0] * NX + d[1] + a1) * UNS + d[2] * UJ + d[3] * n + h * vec) for d in dec]
                cost += phase_cost(ad, w)
                ideal_cost += ideal(ad, w)
        for m1 in range(n):
            ad = [None if d is None else 8 * ((d[0] * TX + d[1]) * WNS + d[2] * WJ + m1 * n + d[3]) for d in dec]
            cost += phase_cost(ad, 8)
            ideal_cost += ideal(ad, 8)
    # x2 loads
    L2 = TY * TX * n * n
    for base in range(0, ((L2 + T - 1) // T) * T, 32):
        dec = []
        for t in range(base, base + 32):
            if t >= L2:
                dec.append(None)
                continue
            dec.append((t % n, (t // n) % TX, (t // (n * TX)) % n, t // (n * TX * n)))
        for a2 in (0, 1):
            for h in range(n // vec):
                ad = [None if d is None else 8 * (((d[3] + a2) * TX + d[1]) * WNS + d[2] * WJ + d[0] * n + h * vec) for d in dec]
                cost += phase_cost(ad, w)
                ideal_cost += ideal(ad, w)
    # x3 stores into V
    L3 = NY * NX * n * n
    for base in range(0, ((L3 + T - 1) // T) * T, 32):
        for m3 in range(n):
            ad = []
            for t in range(base, base + 32):
                if t >= L3:
                    ad.append(None)
                    continue
                col, line = divmod(t, n * n)
                ad.append(8 * (col * UNS + m3 * UJ + line))
            cost += phase_cost(ad, 8)
            ideal_cost += ideal(ad, 8)
    return cost, ideal_cost


def search(N):
    n = N + 1
    best = None
    for pu, pn, pw, pv in itertools.product(range(0, 5), range(0, 5), range(0, 5), range(0, 5)):
        UJ = n * n + pu
        UNS = n * UJ + pn
        WJ = n * n + pw
        WNS = n * WJ + pv
        if n % 2 == 0 and (UJ % 2 or UNS % 2):
            continue  # 16-B vector loads of V lines
        if n % 2 == 0 and (WJ % 2 or WNS % 2):
            continue  # 16-B vector loads of W rows
        c, ic = evaluate(N, UJ, UNS, WJ, WNS)
        smem = 8 * ((TILES[N][0] + 1) * (TILES[N][1] + 1) * UNS + (TILES[N][1] + 1) * TILES[N][0] * WNS)
        key = (c, smem)
        if best is None or key < best[0]:
            best = (key, (UJ, UNS, WJ, WNS), ic)
    return best


if __name__ == "__main__":
    for N in range(6):
        (c, smem), lay, ic = search(N)
        print(f"N={N}: UJ,UNS,WJ,WNS={lay}  wavefronts={c} (ideal {ic})  smem={smem / 1024:.1f} KB")
