"""Search the padded shared-memory strides of a cell (hd_cell.cuh, CellLayout).

A cell's element with digits (d_0, ..., d_{D-1}) sits at sum_i d_i S_i in shared memory. The layout is
ADDITIVE, so a thread's tile element is (its rest offset) + (compile-time constant): the load/store
address is base + immediate, no per-element index arithmetic. The strides are chosen to make the tile
accesses of every phase (and the 16-byte cp.async fill) bank-conflict free where possible:

  * injective: S_i > (N - 1) sum_{j<i} S_j (mixed radix);
  * N even: S_i even for i >= 1 (16-byte pairs along dim 0 stay aligned and contiguous);
  * cost: shared-memory wavefronts of one CTA (256 threads, CT = 256 / N^(D-2) cells) summed over the
    phase tile accesses (64-bit: 16 lanes per wavefront; 128-bit pairs along dim 0 when P = 0 and N
    is even: 8 lanes) and the cp.async fill (128-bit, consecutive pairs).

python tools/smem_layout.py          -> prints the C++ table for hd_cell.cuh and the costs
"""
from __future__ import annotations

import itertools


def phases(D):
    out = []
    for ph in range((D + 1) // 2):
        P = 0 if ph == 0 else 2 * ph - 1
        Q = D - 1 if ph == 0 else 2 * ph
        out.append((P, Q))
    return out


def size_of(S, N):
    return 1 + (N - 1) * sum(S)


def wavefronts(addrs, lanes_per_wf, unit):
    """addrs: per-lane address in doubles (None: inactive); unit: doubles per access."""
    tot = 0
    for s in range(0, len(addrs), lanes_per_wf):
        grp = [a for a in addrs[s:s + lanes_per_wf] if a is not None]
        if not grp:
            continue
        slots = {}
        nslot = 128 // (8 * unit)
        for a in grp:
            key = (a // unit) % nslot
            slots.setdefault(key, set()).add(a // unit)
        tot += max(len(v) for v in slots.values())
    return tot


def cost(S, D, N, phys=None):
    """Wavefronts per CTA of the tile accesses of all phases + the cell fill."""
    NT = N ** (D - 2)
    CT = max(1, 256 // NT)
    nd = N ** D
    ndp = size_of(S, N) if phys is None else nd
    if ndp % 2 and N % 2 == 0:
        ndp += 1
    if phys is None:
        def phys(x):
            p = 0
            for i in range(D):
                p += (x % N) * S[i]
                x //= N
            return p
    total = 0
    nthreads = ((CT * NT + 31) // 32) * 32
    for (P, Q) in phases(D):
        rest = [j for j in range(D) if j not in (P, Q)]
        vec = P == 0 and N % 2 == 0
        for w in range(0, nthreads, 32):
            addrs = []
            for lane in range(32):
                tid = w + lane
                k, r = divmod(tid, NT)
                if k >= CT:
                    addrs.append(None)
                    continue
                x = 0
                for j in rest:
                    x += (r % N) * N ** j
                    r //= N
                addrs.append(k * ndp + phys(x))
            total += wavefronts(addrs, 8, 2) if vec else wavefronts(addrs, 16, 1)
    # fill: consecutive 16-byte pairs (N even) or doubles
    if N % 2 == 0:
        for w in range(0, CT * nd // 2, 32):
            addrs = []
            for lane in range(32):
                e = 2 * (w + lane)
                if e >= CT * nd:
                    addrs.append(None)
                    continue
                kc, x = divmod(e, nd)
                addrs.append(kc * ndp + phys(x))
            total += wavefronts(addrs, 8, 2) / max(1, nd // 64)  # weight: fill is one pass per group
    return total


def xor_phys(D, N):
    def f(x):
        if N == 4 and D >= 4:
            return x ^ (((x >> 6) & 3) << 2) ^ (((x >> 4) & 1) << 1)
        return x
    return f


def search(D, N, span=None, max_growth=1.2):
    """Beam search over the strides S_1..S_{D-1} (S_0 = 1)."""
    span = span if span is not None else 2 * N + 2
    step = 2 if N % 2 == 0 else 1
    beam = [([1], 0.0)]
    for i in range(1, D):
        cand = []
        for S, _ in beam:
            lb = (N - 1) * sum(S) + 1
            if step == 2 and lb % 2:
                lb += 1
            for pad in range(0, span, step):
                S2 = S + [lb + pad]
                # partial cost: remaining strides unpadded continuation
                T = list(S2)
                while len(T) < D:
                    nxt = (N - 1) * sum(T) + 1
                    if step == 2 and nxt % 2:
                        nxt += 1
                    T.append(nxt)
                if size_of(T, N) > max_growth * N ** D and pad > 0:
                    continue  # bounded smem growth
                cand.append((S2, cost(T, D, N) + 1e-3 * size_of(T, N)))
        cand.sort(key=lambda c: c[1])
        beam = cand[:12]
    return beam[0][0]


def built():
    for D in range(2, 7):
        for N in range(2, 7):
            if N ** D > 4096 or N ** (D - 2) > 256:
                continue
            yield D, N


if __name__ == "__main__":
    rows = []
    for D, N in built():
        S = search(D, N)
        base = [N ** i for i in range(D)]
        c_new = cost(S, D, N)
        c_old = cost(base, D, N, phys=xor_phys(D, N))
        c_lin = cost(base, D, N)
        rows.append((D, N, S, size_of(S, N)))
        print(f"// D={D} N={N} S={S} size={size_of(S, N)} (nd {N ** D}) cost {c_new:.1f} "
              f"(xor {c_old:.1f}, plain {c_lin:.1f})")
