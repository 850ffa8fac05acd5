"""Shared-memory bank-conflict model of the Stockham exchanges in
LineFFT::run_f (csrc/kernels/fft_core.cuh) for one warp of a combine kernel
(lanes = (line % (32/T)) * T + j).  64-bit accesses: a warp request is
served in wavefronts of 16 lanes (128 B); inside a half-warp, lanes whose
float2 addresses differ but share a bank pair (addr mod 16) serialise.

    python scripts/tools/bank_sim.py 160        -> wavefronts per line for the
                                                  current layout and the best
                                                  (stride, pad) found
"""
import itertools
import sys


def odd_part(n):
    while n % 2 == 0:
        n //= 2
    return n


def plan(N, RQ=16):
    M = odd_part(N)
    Q = 0 if M == 1 else (4 if N // M >= 4 else N // M)
    R = (RQ if RQ < N else N) if M == 1 else M * Q
    first = R if M == 1 else M
    step = R if M == 1 else Q
    radices, n = [], N
    while n > 1:
        r = (first if first < n else n) if not radices else (step if n >= step else n)
        radices.append(r)
        n //= r
    return R, N // R, radices


def accesses(N, RQ=16):
    """Per exchange round: list of (kind, [per-j float2 index within the line]) warp instructions."""
    R, T, rad = plan(N, RQ)
    ns = [1]
    for r in rad[:-1]:
        ns.append(ns[-1] * r)
    out = []
    for p in range(1, len(rad)):
        Rq, Nq = rad[p - 1], ns[p - 1]
        Sq = R // Rq
        for sc in range(Sq):
            for qc in range(Rq):
                idx = []
                for j in range(T):
                    g = j + sc * T
                    base = (g // Nq) * Nq * Rq + (g % Nq)
                    idx.append(base + qc * Nq)
                out.append(("st", idx))
        for m in range(R):
            out.append(("ld", [j + T * m for j in range(T)]))
    return R, T, out


def wavefronts(addrs):
    w = 0
    for h in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(h):
            banks.setdefault(a % 16, set()).add(a)
        w += max((len(v) for v in banks.values()), default=0)
    return w


def cost(N, stride, pad, RQ=16):
    R, T, acc = accesses(N, RQ)
    lines = max(1, 32 // T)
    tot = {"st": 0, "ld": 0}
    for kind, idx in acc:
        addrs = []
        for L in range(lines):
            for j in range(T):
                if L * T + j < 32:
                    addrs.append(L * stride + pad(idx[j]))
        tot[kind] += wavefronts(addrs[:32])
    ideal = {k: 2 * sum(1 for kk, _ in acc if kk == k) for k in tot}
    return tot, ideal


def cur_pad(p):
    return p + (p >> 4)


def main():
    N = int(sys.argv[1])
    padded = N + (N >> 4)
    cur = padded | 1
    tot, ideal = cost(N, cur, cur_pad)
    print(f"N={N} plan={plan(N)} current stride {cur}: st {tot['st']} ld {tot['ld']} (ideal {ideal['st']} / {ideal['ld']})")
    best = []
    for k, stride_extra in itertools.product(range(0, 7), range(0, 48)):
        pad = (lambda p: p) if k == 0 else (lambda p, k=k: p + (p >> k))
        base = N + (0 if k == 0 else (N - 1 >> k) + 1)
        stride = base + stride_extra
        t, _ = cost(N, stride, pad)
        best.append((t["st"] + t["ld"], k, stride, t))
    best.sort()
    for b in best[:8]:
        print("  pad shift", b[1], "stride", b[2], "st", b[3]["st"], "ld", b[3]["ld"], "total", b[0])


if __name__ == "__main__":
    main()
