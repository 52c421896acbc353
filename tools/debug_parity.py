"""Debug helper: compare one small mesh operator against the oracle and report where it differs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import capi as oracle  # noqa: E402
from paper_2002_08110_b200 import Mesh  # noqa: E402
import test_gpu_parity as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "d4k1vlasov"
spec = dict(T.SMALL)[name]
m = Mesh(spec)
print("traces", m.traces())
N = m.owned_dofs
u = np.random.default_rng(1).uniform(-1, 1, N)
ud = torch.from_numpy(u).cuda()
vd = torch.empty_like(ud)
mode = sys.argv[2] if len(sys.argv) > 2 else "adv"
if mode == "adv":
    m.apply_advection(ud, vd)
    torch.cuda.synchronize()
    got = vd.cpu().numpy()
    ref = oracle.apply_advection(spec, u)
else:
    nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    bufs = [ud, vd, torch.empty_like(ud)]
    dt = 1e-3
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps)
    torch.cuda.synchronize()
    got = bufs[sol].cpu().numpy()
    ref = oracle.rk_steps(spec, u, 0.0, dt, nsteps)
d = spec["d_x"] + spec["d_v"]
nd = (spec["k"] + 1) ** d
err = np.abs(got - ref).reshape(-1, nd).max(axis=1)
print("max err", err.max(), "scale", np.abs(ref).max())
cells = spec["cells"]
bad = np.nonzero(err > 1e-10 * np.abs(ref).max())[0]
print("bad cells", len(bad), "of", len(err))
for c in bad[:20]:
    cc = []
    r = c
    for i in range(d):
        cc.append(r % cells[i])
        r //= cells[i]
    print(c, cc, err[c])
