"""Thin ctypes binding of libhd.so (include/hd.h). Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels. There is no CPU fallback: if libhd.so is missing or
no CUDA device is present the calls raise."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HD_LIB_PATH") or os.path.join(HERE, "libhd.so")

HD_STATUS = {0: "HD_OK", -1: "HD_ERR_ARG", -2: "HD_ERR_UNSUPPORTED", -3: "HD_ERR_CUDA", -4: "HD_ERR_NCCL",
             -5: "HD_ERR_OOM", -6: "HD_ERR_STATE"}
RECIPES = {"gauss2d": 0, "uniform": 1, "sines": 2, "maxwellian": 3}


class HDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{HD_STATUS.get(status, status)}: {msg}")
        self.status = status


class HdMeshDesc(ctypes.Structure):
    _fields_ = [
        ("d_x", ctypes.c_int), ("d_v", ctypes.c_int), ("k", ctypes.c_int),
        ("cells", ctypes.c_longlong * 6), ("lo", ctypes.c_double * 6), ("hi", ctypes.c_double * 6),
        ("a_const", ctypes.c_double * 6), ("a_lin", ctypes.c_double * 36),
        ("flux", ctypes.c_int), ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
        ("nccl_id", ctypes.c_void_p), ("xparts", ctypes.c_int * 3), ("vparts", ctypes.c_int * 3),
    ]


_lib = None

# every symbol include/hd.h declares (checked by tests/test_abi.py)
EXPORTS = ["hd_create_mesh", "hd_destroy_mesh", "hd_mesh_info", "hd_mesh_box", "hd_apply_advection", "hd_apply_advection_fcl", "hd_vp_fields", "hd_apply_advection_vp", "hd_vp_rk_step",
           "hd_basis_change", "hd_apply_advection_gll", "hd_rk_step_gll", "hd_basis_tables",
           "hd_apply_inv_mass", "hd_apply_mass", "hd_rk_step", "hd_rk_stage", "hd_rk_step_host", "hd_apply_advection_group",
           "hd_rk_step_group", "hd_fill_initial", "hd_tables_1d", "hd_lsrk_coefficients", "hd_mesh_traces",
           "hd_nccl_unique_id", "hd_partition_info", "hd_halo_list", "hd_halo_chunks", "hd_launch_count", "hd_last_error"]


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libhd.so not built at {path}; run `python -m paper_2002_08110_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    vp, dp, ll = ctypes.c_void_p, P(ctypes.c_double), ctypes.c_longlong
    lib.hd_create_mesh.argtypes = [P(HdMeshDesc), P(vp)]
    lib.hd_destroy_mesh.argtypes = [vp]
    lib.hd_mesh_info.argtypes = [vp, P(ll), P(ll), P(ll)]
    lib.hd_apply_advection.argtypes = [vp, vp, vp, ctypes.c_double, vp]
    lib.hd_apply_advection_fcl.argtypes = [vp, vp, vp, ctypes.c_double, vp]
    lib.hd_vp_fields.argtypes = [vp, vp, vp, vp, vp]
    lib.hd_apply_advection_vp.argtypes = [vp, vp, vp, vp, vp]
    lib.hd_vp_rk_step.argtypes = [vp, P(vp), ctypes.c_double, ctypes.c_double, ctypes.c_int, vp]
    lib.hd_basis_change.argtypes = [vp, vp, vp, ctypes.c_int, vp]
    lib.hd_apply_advection_gll.argtypes = [vp, vp, vp, vp, ctypes.c_double, vp]
    lib.hd_rk_step_gll.argtypes = [vp, P(vp), P(ctypes.c_int), ctypes.c_double, ctypes.c_double, ctypes.c_int, vp]
    lib.hd_basis_tables.argtypes = [ctypes.c_int, dp, dp]
    lib.hd_apply_inv_mass.argtypes = [vp, vp, vp]
    lib.hd_apply_mass.argtypes = [vp, vp, vp]
    lib.hd_rk_step.argtypes = [vp, P(vp), P(ctypes.c_int), ctypes.c_double, ctypes.c_double, ctypes.c_int, vp]
    lib.hd_rk_stage.argtypes = [vp, vp, vp, vp, ctypes.c_int, ctypes.c_double, vp]
    lib.hd_rk_step_host.argtypes = [vp, vp, vp, P(vp), ctypes.c_double, ctypes.c_double, ctypes.c_int, vp]
    lib.hd_fill_initial.argtypes = [vp, vp, ctypes.c_int, ctypes.c_ulonglong, vp]
    lib.hd_tables_1d.argtypes = [ctypes.c_int, dp, dp, dp, dp, dp]
    lib.hd_lsrk_coefficients.argtypes = [dp, dp]
    lib.hd_mesh_traces.argtypes = [vp, P(ctypes.c_int), P(ctypes.c_int)]
    lib.hd_mesh_box.argtypes = [vp, P(ll), P(ll), P(ctypes.c_int)]
    lib.hd_apply_advection_group.argtypes = [P(vp), ctypes.c_int, P(vp), P(vp), ctypes.c_double, vp]
    lib.hd_rk_step_group.argtypes = [P(vp), ctypes.c_int, P(vp), P(ctypes.c_int), ctypes.c_double,
                                     ctypes.c_double, ctypes.c_int, vp]
    lib.hd_nccl_unique_id.argtypes = [vp]
    lib.hd_partition_info.argtypes = [P(HdMeshDesc), P(ctypes.c_int), P(ll), P(ll)]
    lib.hd_halo_list.argtypes = [P(HdMeshDesc), ctypes.c_int, ctypes.c_int, P(ll), P(ll), P(ctypes.c_int)]
    lib.hd_halo_chunks.argtypes = [P(HdMeshDesc), P(ctypes.c_int), P(ll), P(ll)]
    lib.hd_launch_count.argtypes = [vp]
    lib.hd_launch_count.restype = ll
    lib.hd_last_error.restype = ctypes.c_char_p
    for name in EXPORTS[:-2]:
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(st):
    if st != 0:
        raise HDError(st, load_library().hd_last_error().decode())


def make_desc(spec: dict, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None,
              xparts=None, vparts=None) -> HdMeshDesc:
    ds = HdMeshDesc()
    d = spec["d_x"] + spec["d_v"]
    ds.d_x, ds.d_v, ds.k = spec["d_x"], spec["d_v"], spec["k"]
    for i in range(d):
        ds.cells[i] = int(spec["cells"][i])
        ds.lo[i] = float(spec["lo"][i])
        ds.hi[i] = float(spec["hi"][i])
        ds.a_const[i] = float(spec["a_const"][i])
        lin = spec.get("a_lin")
        if lin is not None:
            for j in range(d):
                ds.a_lin[6 * i + j] = float(lin[i][j])
    ds.flux = {"upwind": 0, "central": 1}[spec.get("flux", "upwind")]
    ds.rank, ds.nranks = rank, nranks
    if xparts is not None:
        for i, p in enumerate(xparts):
            ds.xparts[i] = int(p)
    if vparts is not None:
        for i, p in enumerate(vparts):
            ds.vparts[i] = int(p)
    ds._nccl_buf = None
    if nccl_id is not None:
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        ds._nccl_buf = buf
        ds.nccl_id = ctypes.cast(buf, ctypes.c_void_p)
    return ds


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it and broadcasts it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().hd_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def partition_info(spec: dict, rank: int, nranks: int, xparts=None, vparts=None):
    """Host-only: (xparts[3], box offset[d], box length[d]) of a rank (no GPU needed)."""
    d = spec["d_x"] + spec["d_v"]
    ds = make_desc(spec, rank, nranks, None, xparts, vparts)
    xp, off, ln = (ctypes.c_int * 3)(), (ctypes.c_longlong * 6)(), (ctypes.c_longlong * 6)()
    _check(load_library().hd_partition_info(ctypes.byref(ds), xp, off, ln))
    return list(xp), list(off)[:d], list(ln)[:d]


def halo_list(spec: dict, rank: int, nranks: int, dim: int, which: int, xparts=None, vparts=None):
    """Host-only halo plan query (include/hd.h hd_halo_list): (peer, [global cell ids])."""
    ds = make_desc(spec, rank, nranks, None, xparts, vparts)
    lib = load_library()
    cnt, peer = ctypes.c_longlong(0), ctypes.c_int(0)
    _check(lib.hd_halo_list(ctypes.byref(ds), dim, which, None, ctypes.byref(cnt), ctypes.byref(peer)))
    ids = (ctypes.c_longlong * max(1, cnt.value))()
    _check(lib.hd_halo_list(ctypes.byref(ds), dim, which, ids, ctypes.byref(cnt), ctypes.byref(peer)))
    return peer.value, list(ids)[:cnt.value]


def halo_chunks(spec: dict, rank: int, nranks: int, xparts=None, vparts=None):
    """Host-only v-chunk plan (include/hd.h hd_halo_chunks): (chunk unit bounds, per chunk a dict per x dim:
    sr, sl ((first entry of hd_halo_list which 1 / 0, count): traces to the right / left rank), rl, rr ((first
    slot, count) from the left / right rank))."""
    ds = make_desc(spec, rank, nranks, None, xparts, vparts)
    lib = load_library()
    nc = ctypes.c_int(0)
    units = (ctypes.c_longlong * 9)()
    plan = (ctypes.c_longlong * (8 * 6 * 8))()
    _check(lib.hd_halo_chunks(ctypes.byref(ds), ctypes.byref(nc), units, plan))
    out = []
    for c in range(nc.value):
        dims = []
        for i in range(6):
            q = plan[(c * 6 + i) * 8:(c * 6 + i + 1) * 8]
            dims.append(dict(sr=(q[0], q[1]), sl=(q[2], q[3]), rl=(q[4], q[5]), rr=(q[6], q[7])))
        out.append(dims)
    return list(units)[:nc.value + 1], out


def tables_1d(n: int):
    """Host-side 1D tables of the product path (no GPU needed)."""
    import numpy as np
    xi, w = np.zeros(n), np.zeros(n)
    K, lam, tau = np.zeros((2, n, n)), np.zeros((2, n)), np.zeros((2, n))
    P = ctypes.POINTER(ctypes.c_double)
    _check(load_library().hd_tables_1d(n, *[a.ctypes.data_as(P) for a in (xi, w, K, lam, tau)]))
    return dict(xi=xi, w=w, K=K, lam=lam, tau=tau)


def basis_tables(n: int):
    """Host-side GLL points and the four basis-change matrices [kind][out][in] (hd.h hd_basis_tables)."""
    import numpy as np
    gll, T = np.zeros(n), np.zeros((4, n, n))
    P = ctypes.POINTER(ctypes.c_double)
    _check(load_library().hd_basis_tables(n, gll.ctypes.data_as(P), T.ctypes.data_as(P)))
    return gll, T


def lsrk_coefficients():
    import numpy as np
    a, b = np.zeros(5), np.zeros(5)
    P = ctypes.POINTER(ctypes.c_double)
    _check(load_library().hd_lsrk_coefficients(a.ctypes.data_as(P), b.ctypes.data_as(P)))
    return a, b


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class Mesh:
    """A mesh of the C ABI. Vectors are torch float64 CUDA tensors of ``owned_dofs`` elements."""

    def __init__(self, spec: dict, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None, xparts=None,
                 vparts=None):
        lib = load_library()
        self.spec = spec
        self.rank, self.nranks = rank, nranks
        self._desc = make_desc(spec, rank, nranks, nccl_id, xparts, vparts)
        h = ctypes.c_void_p()
        _check(lib.hd_create_mesh(ctypes.byref(self._desc), ctypes.byref(h)))
        self._h = h
        od, b, e = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_longlong()
        _check(lib.hd_mesh_info(h, ctypes.byref(od), ctypes.byref(b), ctypes.byref(e)))
        self.owned_dofs, self.cx_begin, self.cx_end = od.value, b.value, e.value
        d = spec["d_x"] + spec["d_v"]
        off, ln, xp = (ctypes.c_longlong * 6)(), (ctypes.c_longlong * 6)(), (ctypes.c_int * 3)()
        _check(lib.hd_mesh_box(h, off, ln, xp))
        self.box_off, self.box_len, self.xparts = list(off)[:d], list(ln)[:d], list(xp)

    def close(self):
        if getattr(self, "_h", None):
            load_library().hd_destroy_mesh(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _vec(self, x, name):
        import torch
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
                and x.numel() == self.owned_dofs):
            raise ValueError(f"{name} must be a contiguous float64 CUDA tensor of {self.owned_dofs} elements")
        if x.data_ptr() % 16:
            raise ValueError(f"{name} must be 16-byte aligned (hd.h)")
        return ctypes.c_void_p(x.data_ptr())

    def apply_advection(self, u, v, t: float = 0.0, stream=None):
        _check(load_library().hd_apply_advection(self._h, self._vec(u, "u"), self._vec(v, "v"), float(t),
                                                 _stream_handle(stream)))
        return v

    def apply_advection_fcl(self, u, v, t: float = 0.0, stream=None):
        """v <- A(u) through the face-centric loop comparison path (hd.h hd_apply_advection_fcl)."""
        _check(load_library().hd_apply_advection_fcl(self._h, self._vec(u, "u"), self._vec(v, "v"), float(t),
                                                     _stream_handle(stream)))
        return v

    def _field(self, x, count, name):
        import torch
        if x is None:
            return None
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
                and x.numel() == count):
            raise ValueError(f"{name} must be a contiguous float64 CUDA tensor of {count} elements")
        return ctypes.c_void_p(x.data_ptr())

    def vp_sizes(self):
        """(x nodes = ncx * n^d_x, E doubles = d_x * x nodes) of a Vlasov-Poisson mesh."""
        n = self.spec["k"] + 1
        nxn = 1
        for c in self.spec["cells"][: self.spec["d_x"]]:
            nxn *= c * n
        return nxn, self.spec["d_x"] * nxn

    def vp_fields(self, f, rho=None, E=None, stream=None):
        """rho = 1 - int f dv and E = -grad phi at the x nodes (hd.h hd_vp_fields)."""
        nxn, ne = self.vp_sizes()
        _check(load_library().hd_vp_fields(self._h, self._vec(f, "f"), self._field(rho, nxn, "rho"),
                                           self._field(E, ne, "E"), _stream_handle(stream)))
        return rho, E

    def apply_advection_vp(self, u, E, v, stream=None):
        """v <- A(u) with a = (v, -E(x)) (hd.h hd_apply_advection_vp)."""
        _check(load_library().hd_apply_advection_vp(self._h, self._vec(u, "u"), self._field(E, self.vp_sizes()[1], "E"),
                                                    self._vec(v, "v"), _stream_handle(stream)))
        return v

    def vp_rk_step(self, bufs, t: float, dt: float, nsteps: int = 1, stream=None):
        """nsteps Vlasov-Poisson LSRK(5,4) steps; bufs[0] = f updated in place (hd.h hd_vp_rk_step)."""
        arr = (ctypes.c_void_p * 3)(*[self._vec(b, "buf") for b in bufs])
        _check(load_library().hd_vp_rk_step(self._h, arr, float(t), float(dt), int(nsteps), _stream_handle(stream)))
        return bufs[0]

    def apply_inv_mass(self, u, stream=None):
        _check(load_library().hd_apply_inv_mass(self._h, self._vec(u, "u"), _stream_handle(stream)))
        return u

    def apply_mass(self, u, stream=None):
        _check(load_library().hd_apply_mass(self._h, self._vec(u, "u"), _stream_handle(stream)))
        return u

    def rk_step(self, bufs, sol: int, t: float, dt: float, nsteps: int = 1, stream=None) -> int:
        arr = (ctypes.c_void_p * 3)(*[self._vec(b, f"buf[{i}]").value for i, b in enumerate(bufs)])
        s = ctypes.c_int(sol)
        _check(load_library().hd_rk_step(self._h, arr, ctypes.byref(s), float(t), float(dt), int(nsteps),
                                         _stream_handle(stream)))
        return s.value

    BASIS_KINDS = {"gll_to_gauss": 0, "gauss_to_gll": 1, "gll_to_gauss_T": 2, "gauss_to_gll_T": 3}

    def basis_change(self, u, v, kind, stream=None):
        """v <- (S x ... x S) u per cell (hd.h hd_basis_change); v may be u."""
        k = self.BASIS_KINDS[kind] if isinstance(kind, str) else int(kind)
        _check(load_library().hd_basis_change(self._h, self._vec(u, "u"), self._vec(v, "v"), k, _stream_handle(stream)))
        return v

    def apply_advection_gll(self, u, v, work, t: float = 0.0, stream=None):
        """v <- T^T A(T u): the weak form in the GLL basis (hd.h hd_apply_advection_gll)."""
        _check(load_library().hd_apply_advection_gll(self._h, self._vec(u, "u"), self._vec(v, "v"),
                                                     self._vec(work, "work"), float(t), _stream_handle(stream)))
        return v

    def rk_step_gll(self, bufs, sol: int, t: float, dt: float, nsteps: int = 1, stream=None) -> int:
        arr = (ctypes.c_void_p * 3)(*[self._vec(b, f"buf[{i}]").value for i, b in enumerate(bufs)])
        s = ctypes.c_int(sol)
        _check(load_library().hd_rk_step_gll(self._h, arr, ctypes.byref(s), float(t), float(dt), int(nsteps),
                                             _stream_handle(stream)))
        return s.value

    def rk_stage(self, U, dU, out, stage: int, dt: float, stream=None):
        """One fused LSRK stage (0..4): dU <- A_s dU + dt M^-1 A(U); out <- U + B_s dU."""
        _check(load_library().hd_rk_stage(self._h, self._vec(U, "U"), self._vec(dU, "dU"), self._vec(out, "out"),
                                          int(stage), float(dt), _stream_handle(stream)))

    def rk_step_host(self, u_host, u_out_host, dbufs, t: float, dt: float, nsteps: int = 1, stream=None):
        import torch
        for x in (u_host, u_out_host):
            if not (isinstance(x, torch.Tensor) and not x.is_cuda and x.dtype == torch.float64
                    and x.is_contiguous() and x.numel() == self.owned_dofs):
                raise ValueError("host buffers must be contiguous float64 CPU tensors of owned_dofs elements")
        arr = (ctypes.c_void_p * 3)(*[self._vec(b, f"dbuf[{i}]").value for i, b in enumerate(dbufs)])
        _check(load_library().hd_rk_step_host(self._h, ctypes.c_void_p(u_host.data_ptr()),
                                              ctypes.c_void_p(u_out_host.data_ptr()), arr, float(t), float(dt),
                                              int(nsteps), _stream_handle(stream)))
        return u_out_host

    def fill_initial(self, u, recipe: str, seed: int, stream=None):
        _check(load_library().hd_fill_initial(self._h, self._vec(u, "u"), RECIPES[recipe], int(seed),
                                              _stream_handle(stream)))
        return u

    def traces(self):
        d = self.spec["d_x"] + self.spec["d_v"]
        tm, rs = (ctypes.c_int * 6)(), (ctypes.c_int * 6)()
        _check(load_library().hd_mesh_traces(self._h, tm, rs))
        return list(tm)[:d], list(rs)[:d]

    @property
    def launch_count(self) -> int:
        return int(load_library().hd_launch_count(self._h))


def apply_advection_group(meshes, us, vs, t: float = 0.0, stream=None):
    """Loopback multi-rank v <- A(u): meshes[r] is rank r of P (no NCCL), all on the current device."""
    P = len(meshes)
    ms = (ctypes.c_void_p * P)(*[m._h.value for m in meshes])
    ua = (ctypes.c_void_p * P)(*[m._vec(u, "u").value for m, u in zip(meshes, us)])
    va = (ctypes.c_void_p * P)(*[m._vec(v, "v").value for m, v in zip(meshes, vs)])
    _check(load_library().hd_apply_advection_group(ms, P, ua, va, float(t), _stream_handle(stream)))


def rk_step_group(meshes, bufs, sol: int, t: float, dt: float, nsteps: int = 1, stream=None) -> int:
    """Loopback multi-rank LSRK steps; bufs[r] = the 3 buffers of rank r. Returns the new sol."""
    P = len(meshes)
    ms = (ctypes.c_void_p * P)(*[m._h.value for m in meshes])
    flat = [m._vec(b, "buf").value for m, bs in zip(meshes, bufs) for b in bs]
    arr = (ctypes.c_void_p * (3 * P))(*flat)
    s = ctypes.c_int(sol)
    _check(load_library().hd_rk_step_group(ms, P, arr, ctypes.byref(s), float(t), float(dt), int(nsteps),
                                           _stream_handle(stream)))
    return s.value
