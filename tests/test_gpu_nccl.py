"""GPU, >= 2 devices: the NCCL transport of the v-chunk pipelined halo -- two processes, one
GPU each, ncclUniqueId broadcast over torch.distributed -- equals one rank BITWISE (C18) for apply_advection
and 3 LSRK steps. Skipped on a one-GPU box (the loopback tests in test_gpu_multirank.py run the same chunk
plan, buffers and kernels there)."""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _spec():
    d_x, d_v = 3, 2
    d = d_x + d_v
    lin = [[0.0] * d for _ in range(d)]
    lin[0][3] = lin[1][4] = 1.0
    return dict(d_x=d_x, d_v=d_v, k=3, cells=[6, 8, 4, 4, 4], lo=[0.0] * 3 + [-2.0] * 2, hi=[1.0] * 3 + [2.0] * 2,
                a_const=[0.0, 0.0, 0.5, 0.3, -0.2], a_lin=lin, flux="upwind")


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    from paper_2002_08110_b200 import Mesh, _binding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    t = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        t.copy_(torch.tensor(list(_binding.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    spec = _spec()
    m = Mesh(spec, rank=rank, nranks=world, nccl_id=bytes(t.cpu().tolist()), xparts=[1, 1, world])
    d = 5
    nd = 4 ** d
    u = np.random.default_rng(5).uniform(-1, 1, int(np.prod(spec["cells"])) * nd)
    cv = u.reshape(list(spec["cells"][::-1]) + [nd])
    box = tuple(slice(m.box_off[i], m.box_off[i] + m.box_len[i]) for i in reversed(range(d)))
    ul = torch.from_numpy(np.ascontiguousarray(cv[box]).reshape(-1)).cuda()
    v = torch.empty_like(ul)
    m.apply_advection(ul, v)
    bufs = [ul.clone(), torch.empty_like(ul), torch.empty_like(ul)]
    sol = m.rk_step(bufs, 0, 0.0, 1e-3, 3)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"a{rank}.npy"), v.cpu().numpy())
    np.save(os.path.join(outdir, f"rk{rank}.npy"), bufs[sol].cpu().numpy())
    np.save(os.path.join(outdir, f"box{rank}.npy"), np.array(m.box_off + m.box_len))
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs (NCCL ranks must not share a device)")
def test_nccl_two_ranks_equal_single_rank():
    import torch
    import torch.multiprocessing as mp
    from paper_2002_08110_b200 import Mesh
    spec = _spec()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(2, port, td), nprocs=2, join=True)
        d = 5
        nd = 4 ** d
        u = np.random.default_rng(5).uniform(-1, 1, int(np.prod(spec["cells"])) * nd)
        one = Mesh(spec)
        ud = torch.from_numpy(u).cuda()
        vd = torch.empty_like(ud)
        one.apply_advection(ud, vd)
        bufs = [ud.clone(), torch.empty_like(ud), torch.empty_like(ud)]
        sol = one.rk_step(bufs, 0, 0.0, 1e-3, 3)
        ref_a = vd.cpu().numpy().reshape(list(spec["cells"][::-1]) + [nd])
        ref_rk = bufs[sol].cpu().numpy().reshape(ref_a.shape)
        for r in range(2):
            b = np.load(os.path.join(td, f"box{r}.npy"))
            box = tuple(slice(b[i], b[i] + b[d + i]) for i in reversed(range(d)))
            assert np.array_equal(np.load(os.path.join(td, f"a{r}.npy")), ref_a[box].reshape(-1))
            assert np.array_equal(np.load(os.path.join(td, f"rk{r}.npy")), ref_rk[box].reshape(-1))
