"""Search the K order (which (vertex a, component j) each lane q reads at k-step ks) of the m=5
fused cell-pair kernel's passes that minimises shared-memory wavefronts: a half-warp (16 lanes =
4 lines g x 4 k-lanes q) issues one 8-byte load; its wavefront count is the largest number of
distinct addresses that fall on one of the 16 double-wide bank pairs.  The order within a k-step
does not matter, only the partition of the 12 (a, j) inputs into 3 k-steps."""
import itertools

n, TX, TY, NY = 6, 4, 4, 5
n2 = n * n
WM, WCS = n2 + 1, n * (n2 + 1)          # W [row][cell][m1][j3 j2]
VJ, VCS = n2 + 1, n * (n2 + 1)          # V [cell][j3][m2 m1]
PAIRS = [(a, j) for a in (0, 1) for j in range(n)]


def wavefronts(addrs):
    banks = {}
    for x in set(addrs):
        banks.setdefault(x % 16, set()).add(x)
    return max(len(v) for v in banks.values())


def lines(L, groups):
    for G in range(groups):
        for half in (0, 1):
            yield [min(G * 8 + half * 4 + g, L - 1) for g in range(4)]


def cost(partition, line_addr, k_addr, L):
    groups = (L + 7) // 8
    total = 0
    for ls in lines(L, groups):
        for ks_set in partition:
            total += wavefronts([line_addr(l) + k_addr(a, j) for l in ls for (a, j) in ks_set])
    return total


def x2_line(l):
    cell, r = divmod(l, n2)
    j3, m1 = divmod(r, n)
    return cell * WCS + m1 * WM + j3 * n


def x2_k(a, j):
    return a * TX * WCS + j


def x3_line(l):
    cell, r = divmod(l, n2)
    return cell * VCS + r


def x3_k(a, j):
    return j * VJ  # the plane (a) selects a buffer whose offset is 0 mod 16 doubles


def partitions():
    for A in itertools.combinations(PAIRS, 4):
        if (0, 0) not in A:
            continue
        rest = [p for p in PAIRS if p not in A]
        for B in itertools.combinations(rest, 4):
            if rest[0] not in B:
                continue
            C = tuple(p for p in rest if p not in B)
            yield (A, B, C)


natural = tuple(tuple(PAIRS[4 * ks + q] for q in range(4)) for ks in range(3))
for name, la, ka, L in (("x2", x2_line, x2_k, TY * TX * n2), ("x3", x3_line, x3_k, TY * TX * n2)):
    base = cost(natural, la, ka, L)
    best = min(partitions(), key=lambda p: cost(p, la, ka, L))
    print(name, "natural", base, "best", cost(best, la, ka, L), best)


# ---- the m=5 reconstruction (rcp::Cfg<5, 4, 2, 2>): one K order shared by its three passes
# (all of them contract with the same H, so one set of B fragments) --------------------------
RTX, RTY, RNX, RNY = 4, 2, 5, 3
S = 2 * n
UNS = n ** 3
RWI, RWCS = n2 + 1, S * (n2 + 1)   # W [row][cell][i1][j3 j2]
RVJ, RVCS = S * S + 4, n * (S * S + 4)  # V [cell][j3][i2 i1]


def r1_line(l):
    rc, jj = divmod(l, n2)
    ly, cx = divmod(rc, RTX)
    return (ly * RNX + cx) * UNS + jj * n


def r1_k(a, j):
    return a * UNS + j


def r2_line(l):
    cell, r = divmod(l, n * S)
    j3, i1 = divmod(r, S)
    return cell * RWCS + i1 * RWI + j3 * n


def r2_k(a, j):
    return a * RTX * RWCS + j


def r3_line(l):
    cell, r = divmod(l, S * S)
    return cell * RVCS + r


def r3_k(a, j):
    return j * RVJ


def recon_cost(p):
    return (cost(p, r1_line, r1_k, RNY * RTX * n2) + cost(p, r2_line, r2_k, RTY * RTX * n * S)
            + cost(p, r3_line, r3_k, RTY * RTX * S * S))


if __name__ == "__main__":
    base = recon_cost(natural)
    best = min(partitions(), key=recon_cost)
    print("recon natural", base, "best", recon_cost(best), best)
