"""Multi-rank host logic on the CPU: the x-space partition and the halo
plan of include/hd.h (hd_partition_info, hd_halo_list), which need no GPU.

* every cell is owned by exactly one rank and v-cells are never split (v part undivided);
* the traces rank r sends to rank q are exactly, and in the same order, those q expects from r -- checked
  across real processes: world_size-2 ``gloo`` groups exchange their plans with all_gather_object;
* the union of the receive lists is exactly the set of (cell, dim) pairs whose UPWIND neighbour (sign
  of a_i at the cell centre, C3/C11) is owned by another rank -- recomputed here independently with numpy.
"""
import itertools
import os
import socket

import numpy as np
import pytest

from paper_2002_08110_b200 import configs, halo_list, partition_info


def _spec(d_x, d_v, k, cells, lo, hi, a_const, a_lin=None):
    d = d_x + d_v
    if a_lin is None:
        a_lin = [[0.0] * d for _ in range(d)]
    return dict(d_x=d_x, d_v=d_v, k=k, cells=list(cells), lo=list(lo), hi=list(hi), a_const=list(a_const),
                a_lin=[list(r) for r in a_lin], flux="upwind")


def _vlasov(d_x, d_v, cells, k=1):
    d = d_x + d_v
    lin = [[0.0] * d for _ in range(d)]
    for i in range(min(d_x, d_v)):
        lin[i][d_x + i] = 1.0
    ac = [0.0] * d_x + [0.3, -0.2, 0.1][:d_v]
    lo = [0.0] * d_x + [-2.0] * d_v
    hi = [1.0] * d_x + [2.0] * d_v
    return _spec(d_x, d_v, k, cells, lo, hi, ac, lin)


# (name, spec, P, xparts, vparts): automatic x partitions, explicit x-blocks, and checkerboard x-v
# partitions that also split v dims (NEXT-4)
CASES = [
    ("3d-const-P2", _spec(2, 1, 2, [4, 6, 3], [0] * 3, [1] * 3, [1.0, -0.7, 0.3]), 2, None, None),
    ("4d-vlasov-P2", _vlasov(2, 2, [4, 6, 2, 4]), 2, None, None),
    ("4d-vlasov-P4", _vlasov(2, 2, [4, 6, 2, 4]), 4, None, None),
    ("5d-vlasov-P8", _vlasov(3, 2, [4, 4, 6, 2, 2]), 8, None, None),
    ("5d-vlasov-P4-x0split", _vlasov(3, 2, [4, 4, 6, 2, 2]), 4, [4, 1, 1], None),
    ("6d-vlasov-P8", _vlasov(3, 3, [2, 2, 2, 2, 2, 2]), 8, None, None),
    ("4d-vlasov-P4-xv", _vlasov(2, 2, [4, 6, 2, 4]), 4, [2, 1], [1, 2]),
    ("5d-vlasov-P4-v", _vlasov(3, 2, [4, 4, 6, 2, 2]), 4, [1, 1, 1], [2, 2]),
    ("6d-vlasov-P8-xv", _vlasov(3, 3, [2, 2, 2, 2, 2, 2]), 8, [1, 1, 2], [2, 2, 1]),
]


def _sign(spec, i, c):
    """1 if a_i < 0 at the centre of the cell with global coordinates c (reading C11)."""
    d = spec["d_x"] + spec["d_v"]
    h = [(spec["hi"][j] - spec["lo"][j]) / spec["cells"][j] for j in range(d)]
    a = spec["a_const"][i] + sum(spec["a_lin"][i][j] * (spec["lo"][j] + (c[j] + 0.5) * h[j]) for j in range(d))
    return 1 if a < 0 else 0


def _owner_map(spec, P, xparts, vparts=None):
    d = spec["d_x"] + spec["d_v"]
    owner = -np.ones(spec["cells"][::-1], dtype=np.int64).transpose()  # index [c0, c1, ...]
    for r in range(P):
        _, off, ln = partition_info(spec, r, P, xparts, vparts)
        sl = tuple(slice(off[i], off[i] + ln[i]) for i in range(d))
        assert np.all(owner[sl] == -1), "cells owned twice"
        owner[sl] = r
    assert np.all(owner >= 0), "cells owned by nobody"
    return owner


def _gid(spec, c):
    g, s = 0, 1
    for i, ci in enumerate(c):
        g += ci * s
        s *= spec["cells"][i]
    return g


@pytest.mark.parametrize("name,spec,P,xparts,vparts", CASES, ids=[c[0] for c in CASES])
def test_partition_covers_and_halo_is_the_remote_upwind_set(name, spec, P, xparts, vparts):
    d, d_x = spec["d_x"] + spec["d_v"], spec["d_x"]
    owner = _owner_map(spec, P, xparts, vparts)
    xp, off, ln = partition_info(spec, 0, P, xparts, vparts)
    parts = [spec["cells"][i] // ln[i] for i in range(d)]
    assert int(np.prod(parts)) == P
    for i in range(d_x, d):
        want = 1 if vparts is None else vparts[i - d_x]
        assert parts[i] == want, "v dims are split exactly as requested"
    # independent: (cell, dim) pairs whose upwind neighbour is remote, per receiving rank
    expect = {r: set() for r in range(P)}
    for c in itertools.product(*[range(n) for n in spec["cells"]]):
        for i in range(d):
            up = 1 if _sign(spec, i, c) else -1
            cn = list(c)
            cn[i] = (c[i] + up) % spec["cells"][i]
            if owner[tuple(cn)] != owner[c]:
                expect[owner[c]].add((_gid(spec, c), i, owner[tuple(cn)]))
    for r in range(P):
        got = set()
        for i in range(d):
            for which in (2, 3):
                peer, ids = halo_list(spec, r, P, i, which, xparts, vparts)
                assert len(ids) == len(set(ids))
                got |= {(g, i, peer) for g in ids}
        assert got == expect[r], f"rank {r}: halo receive set differs from the remote-upwind set"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, cases, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        errors = []
        for name, spec, P, xparts, vparts in cases:
            d = spec["d_x"] + spec["d_v"]
            # this process plays ranks rank, rank + world, ... of the P-rank partition
            mine = {}
            for r in range(rank, P, world):
                for i in range(d):
                    for which in range(4):
                        mine[(r, i, which)] = halo_list(spec, r, P, i, which, xparts, vparts)
            allp = [None] * world
            dist.all_gather_object(allp, mine)
            plan = {}
            for part in allp:
                plan.update(part)
            for r in range(rank, P, world):
                for i in range(d):
                    # what r receives from its left (which 2) is what the left rank sends right (which 1)
                    for recv_w, send_w in ((2, 1), (3, 0)):
                        peer, rids = plan[(r, i, recv_w)]
                        if peer < 0:
                            continue
                        back, sids = plan[(peer, i, send_w)]
                        if back != r or sids != rids:
                            errors.append(f"{name}: rank {r} dim {i} which {recv_w} vs rank {peer}")
        q.put((rank, errors))
    finally:
        dist.destroy_process_group()


def test_halo_plans_match_across_gloo_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errors in res:
        assert not errors, errors


def test_config_partitions():
    """The bench configs shard as documented: 6D/5D over 2/4/8 ranks (x-slab when it divides)."""
    for name in ("5d", "6d"):
        spec = configs.CONFIGS[name]["spec"]
        for P in (2, 4, 8):
            xp, off, ln = partition_info(spec, P - 1, P)
            assert int(np.prod(xp)) == P
            assert all(spec["cells"][i] % xp[i] == 0 for i in range(3))
        # 2 ranks split the slowest x dim (x-slab)
        assert partition_info(spec, 0, 2)[0] == [1, 1, 2]


# ---- the v-chunk pipeline: real per-chunk messages between gloo processes
CHUNK_CASES = [
    ("5d-pencil-P2-slab", _vlasov(3, 2, [6, 4, 4, 4, 4], k=3), 2, [1, 1, 2], None),
    ("6d-pencil-P2", _vlasov(3, 3, [2, 2, 4, 2, 2, 4], k=3), 2, None, None),
    ("5d-pencil-P4-xblocks", _vlasov(3, 2, [6, 4, 4, 4, 4], k=3), 4, [1, 2, 2], None),
    ("5d-pencil-P4-xv", _vlasov(3, 2, [6, 4, 4, 4, 4], k=3), 4, [1, 1, 2], [2, 1]),
]


def _chunk_worker(rank, world, port, case, q):
    """Rank `rank` of `world`: per v-chunk and x dim, send to each neighbour the global ids of the cells its
    traces are meant for (the chunk's range of the send lists) and check that what arrives from each
    neighbour is exactly the ids of this rank's receive slots of that chunk, and that the chunks partition
    the send lists."""
    import torch
    import torch.distributed as dist
    from paper_2002_08110_b200 import halo_chunks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    errors = []
    try:
        name, spec, P, xparts, vparts = case
        d = spec["d_x"] + spec["d_v"]
        units, chunks = halo_chunks(spec, rank, P, xparts, vparts)
        if len(chunks) < 2:
            errors.append(f"{name}: expected several chunks, got {len(chunks)}")
        lists = {}
        for i in range(d):
            for which in range(4):
                lists[(i, which)] = halo_list(spec, rank, P, i, which, xparts, vparts)
        nleft = {i: len(lists[(i, 2)][1]) for i in range(d)}
        covered_r = {i: [] for i in range(d)}
        covered_l = {i: [] for i in range(d)}
        for c, plan in enumerate(chunks):
            reqs, checks = [], []
            for i in range(d):
                pr, to_right = lists[(i, 1)]
                pl, to_left = lists[(i, 0)]
                if pr < 0:
                    continue
                pi = plan[i]
                (r0, nr), (l0, nl) = pi["sr"], pi["sl"]
                sr = torch.tensor(to_right[r0:r0 + nr], dtype=torch.int64)
                sl = torch.tensor(to_left[l0:l0 + nl], dtype=torch.int64)
                covered_r[i] += list(range(r0, r0 + nr))
                covered_l[i] += list(range(l0, l0 + nl))
                _, from_left = lists[(i, 2)]
                _, from_right = lists[(i, 3)]
                (a, na), (b, nb) = pi["rl"], pi["rr"]
                exp_l = from_left[a:a + na]
                exp_r = from_right[b - nleft[i]:b - nleft[i] + nb]
                rl = torch.empty(na, dtype=torch.int64)
                rr = torch.empty(nb, dtype=torch.int64)
                # one tag per (chunk, dim, direction); the counts agree on both sides by construction
                if sr.numel():
                    reqs.append(dist.isend(sr, pr, tag=c * 16 + i * 2))
                if sl.numel():
                    reqs.append(dist.isend(sl, pl, tag=c * 16 + i * 2 + 1))
                if na:
                    reqs.append(dist.irecv(rl, lists[(i, 2)][0], tag=c * 16 + i * 2))
                if nb:
                    reqs.append(dist.irecv(rr, lists[(i, 3)][0], tag=c * 16 + i * 2 + 1))
                checks.append((i, rl, exp_l, rr, exp_r))
            for r in reqs:
                r.wait()
            for i, rl, exp_l, rr, exp_r in checks:
                if rl.tolist() != list(exp_l) or rr.tolist() != list(exp_r):
                    errors.append(f"{name}: rank {rank} chunk {c} dim {i}: received ids differ")
        for i in range(d):
            if lists[(i, 1)][0] >= 0 and (sorted(covered_r[i]) != list(range(len(lists[(i, 1)][1]))) or
                                          sorted(covered_l[i]) != list(range(len(lists[(i, 0)][1])))):
                errors.append(f"{name}: rank {rank} dim {i}: the chunks do not partition the send lists")
    except Exception as ex:  # noqa: BLE001
        errors.append(f"{case[0]}: rank {rank}: {ex!r}")
    finally:
        q.put((rank, errors))
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CHUNK_CASES, ids=[c[0] for c in CHUNK_CASES])
def test_chunked_halo_messages_between_gloo_ranks(case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = case[2]
    procs = [ctx.Process(target=_chunk_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errors in res:
        assert not errors, errors
