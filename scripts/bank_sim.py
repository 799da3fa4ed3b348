"""Offline shared-memory bank-conflict simulator for the Stockham exchange (graf_fft.cuh).

Plans follow graf_fft.cuh: radices RM, RM, ..., remainder LAST, RM = min(E, RMAX).
Padding: element y lives at y + (y >> sh).  Prints (mean, worst) conflict degree per
(pad shift) for each (M, E, RMAX); 1.0 = conflict-free (8-byte elements, 16 per phase).
"""


def radices(M, E, rmax):
    RM = min(E, rmax)
    r, m = [], M
    while m >= RM:
        r.append(RM)
        m //= RM
    return r + ([m] if m > 1 else [])


def degree(addrs):
    worst = 0
    for ph in range(0, len(addrs), 16):
        b = {}
        for a in set(addrs[ph:ph + 16]):
            b.setdefault(a % 16, set()).add(a)
        worst = max(worst, max(len(v) for v in b.values()))
    return worst


def sim(M, E, sh, rmax):
    def pad(y):
        return y >> sh
    T = M // E
    rad = radices(M, E, rmax)
    tot = cnt = worst = 0
    Ns = 1
    stride = M + (M >> sh)
    for p, R in enumerate(rad[:-1]):
        Q = E // R
        for q in range(Q):
            for r in range(R):
                addrs = []
                for lane in range(32):
                    sl = lane // T if T < 32 else 0
                    t = lane % T if T < 32 else lane
                    jp = t + q * T
                    y = (jp // Ns) * Ns * R + (jp % Ns) + r * Ns
                    addrs.append(sl * stride + pad(y) + y)
                d = degree(addrs)
                tot, cnt, worst = tot + d, cnt + 1, max(worst, d)
        for e in range(E):
            addrs = []
            for lane in range(32):
                sl = lane // T if T < 32 else 0
                t = lane % T if T < 32 else lane
                y = t + e * T
                addrs.append(sl * stride + pad(y) + y)
            d = degree(addrs)
            tot, cnt, worst = tot + d, cnt + 1, max(worst, d)
        Ns *= R
    return (round(tot / cnt, 3) if cnt else 0, worst)


if __name__ == "__main__":
    for M, E, rmax in [(256, 16, 16), (1024, 16, 16), (8192, 16, 16), (1024, 32, 32), (2048, 32, 32),
                       (4096, 32, 32), (8192, 32, 32), (512, 32, 32), (256, 32, 32)]:
        print(M, E, rmax, radices(M, E, rmax), {s: sim(M, E, s, rmax) for s in (3, 4, 5)})
