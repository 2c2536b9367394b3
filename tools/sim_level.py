"""Debug model of ONE partitioning level as the CUDA kernels implement it
(classification tiles, boundaries, stripe fix, sequential permutation agents,
cleanup) -- single-threaded Python, used only to debug index arithmetic on
the CPU.  It is NOT an oracle: parity is always against oracle/."""
import random
import sys


def level(a, splitters_fn, K, B, stripe_elems, tile, agents=3, seed=0):
    n = len(a)
    A = list(a)
    cls = splitters_fn
    nst = (n + stripe_elems - 1) // stripe_elems
    counts, pfill, full, partial = [], [], [], []
    # ---- classify (tile synchronous, same formulas as the kernel)
    for s in range(nst):
        s0 = s * stripe_elems
        s1 = min(n, s0 + stripe_elems)
        buf = [[] for _ in range(K)]
        cnt = [0] * K
        front = 0
        t = s0
        while t < s1:
            c = min(tile, s1 - t)
            items = A[t:t + c]
            b = [cls(x) for x in items]
            tc = [0] * K
            rank = []
            for j in b:
                rank.append(tc[j])
                tc[j] += 1
            nb = [(len(buf[j]) + tc[j]) // B for j in range(K)]
            boff = [0] * K
            acc = 0
            for j in range(K):
                boff[j] = acc
                acc += nb[j]
            nblocks = acc
            # emitted blocks contents
            emit = {}
            for j in range(K):
                stream = list(buf[j])
                for i, x in enumerate(items):
                    if b[i] == j:
                        stream.append(x)
                for q in range(nb[j]):
                    emit[boff[j] + q] = stream[q * B:(q + 1) * B]
                buf[j] = stream[nb[j] * B:]
                cnt[j] += tc[j]
            for g in range(nblocks):
                pos = s0 + (front + g) * B
                assert pos + B <= t + c, "flush overtook the read position"
                A[pos:pos + B] = emit[g]
            front += nblocks
            t += c
        counts.append(cnt)
        pfill.append([len(x) for x in buf])
        full.append(front)
        partial.append(buf)
        # poison the empty tail
        for i in range(s0 + front * B, s1):
            A[i] = None
    # ---- boundaries
    c = [sum(counts[s][j] for s in range(nst)) for j in range(K)]
    f = [sum((counts[s][j] - pfill[s][j]) // B for s in range(nst)) for j in range(K)]
    E = [0]
    for j in range(K):
        E.append(E[-1] + c[j])
    d = [(e + B - 1) // B for e in E]  # region starts in blocks
    SB = stripe_elems // B
    nblk_total = (n + B - 1) // B
    fcum = [0]
    for s in range(nst):
        fcum.append(fcum[-1] + full[s])

    def Fx(x):  # number of full block positions in [0, x)
        cc = x // SB
        if cc >= nst:
            return fcum[nst]
        return fcum[cc] + min(full[cc], x - cc * SB)

    def select(q):  # position of the q-th full block (0-based)
        cc = max(k for k in range(nst) if fcum[k] <= q)
        return cc * SB + (q - fcum[cc])

    fr = [Fx(d[j + 1]) - Fx(d[j]) for j in range(K)]  # full positions in region j
    moves = []
    for s in range(nst):
        c_lo = s * SB
        c_hi = min(c_lo + SB, nblk_total)
        e0 = c_lo + full[s]
        if e0 >= c_hi:
            continue
        for j in range(K):
            r0, r1 = d[j], d[j + 1]
            pe = r0 + fr[j]
            if pe <= e0:
                continue
            if r0 >= c_hi:
                break
            h0, h1 = max(e0, r0), min(c_hi, pe)
            if h0 >= h1:
                continue
            skip = (h0 - r0) - (Fx(h0) - Fx(r0))
            for i in range(h1 - h0):
                g = skip + i
                q = Fx(r1) - g - 1
                moves.append((select(q), h0 + i))
    for src, dst in moves:
        blk = A[src * B:(src + 1) * B]
        assert None not in blk, f"stripe fix moves an empty block {src}->{dst}"
        A[dst * B:(dst + 1) * B] = blk
        A[src * B:(src + 1) * B] = [None] * B
    # check full prefix per region
    for j in range(K):
        for x in range(d[j], d[j] + fr[j]):
            blk = A[x * B:(x + 1) * B]
            assert len(blk) == B and None not in blk, f"bucket {j}: hole at block {x} after stripe fix"
        for x in range(d[j] + fr[j], d[j + 1]):
            blk = A[x * B:(x + 1) * B]
            assert all(v is None for v in blk), f"bucket {j}: full block {x} beyond the prefix"
    # ---- permutation (sequential agents)
    pblk = n // B if n % B else None
    ovf = [None] * B
    w = [d[j] for j in range(K)]
    r = [d[j] + fr[j] - 1 for j in range(K)]

    def get(x):
        return ovf if x == pblk else A[x * B:(x + 1) * B]

    def put(x, blk):
        nonlocal ovf
        if x == pblk:
            ovf = list(blk)
            return "ovf"
        A[x * B:(x + 1) * B] = blk

    ovf_bucket = None
    for ag in range(agents):
        pass
    # single agent sequence
    p = 0
    misses = 0
    while True:
        x = None
        while misses < K:
            if r[p] >= w[p]:
                x = r[p]
                r[p] -= 1
                break
            r[p] -= 1 if False else 0
            p = (p + 1) % K
            misses += 1
        if x is None:
            break
        misses = 0
        buf0 = list(get(x))
        assert None not in buf0, f"read empty block {x}"
        dest = cls(buf0[0])
        while True:
            wo, ro = w[dest], r[dest]
            w[dest] += 1
            if wo <= ro:
                b1 = list(get(wo))
                d2 = cls(b1[0])
                if d2 == dest:
                    continue
                put(wo, buf0)
                buf0, dest = b1, d2
                continue
            if put(wo, buf0) == "ovf":
                ovf_bucket = dest
            break
    for j in range(K):
        assert w[j] == d[j] + f[j], f"bucket {j}: w={w[j]} expected {d[j] + f[j]}"
    # ---- cleanup (phase a: save overlaps + overflow; phase b: fill holes)
    def logical(x, j):
        if ovf_bucket == j and pblk is not None and x >= pblk * B:
            return ovf[x - pblk * B]
        return A[x]
    saved = {}
    for j in range(K):
        W = w[j] * B
        E1 = E[j + 1]
        o0 = max(E1, d[j] * B)
        saved[j] = [logical(x, j) for x in range(o0, W)] if W > o0 else []
        if ovf_bucket == j:
            for x in range(pblk * B, min(E1, n)):
                A[x] = ovf[x - pblk * B]
    for j in range(K):
        E0, E1 = E[j], E[j + 1]
        if E0 == E1:
            continue
        d0 = d[j] * B
        W = w[j] * B
        hd = min(d0, E1)
        tl = max(W, hd)
        holes = list(range(E0, hd)) + (list(range(tl, E1)) if tl < E1 else [])
        srcs = saved[j] + [x for s in range(nst) for x in partial[s][j]]
        assert len(holes) == len(srcs), f"bucket {j}: {len(holes)} holes vs {len(srcs)} sources"
        for h, v in zip(holes, srcs):
            A[h] = v
    assert sorted(A) == sorted(a), "multiset changed"
    for j in range(K):
        assert all(cls(x) == j for x in A[E[j]:E[j + 1]]), f"bucket {j} holds foreign elements"
    return dict(E=E, d=d, f=f, w=w, A=A, ovf=ovf, ovf_bucket=ovf_bucket, partial=partial, pfill=pfill)


if __name__ == "__main__":
    rnd = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
    for trial in range(300):
        n = rnd.randint(1, 3000)
        B = rnd.choice([1, 2, 4, 8, 16])
        K = rnd.choice([2, 4, 8, 16])
        tile = rnd.choice([4, 16, 64, 256])
        se = B * rnd.randint(1, 200)
        a = [rnd.randint(0, 1000) for _ in range(n)]
        spl = sorted(rnd.sample(range(1001), K - 1))

        def cls(x, spl=spl):
            return sum(1 for s in spl if s < x)

        level(a, cls, K, B, se, tile)
    print("ok")
