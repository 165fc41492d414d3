"""Thin ctypes binding of libhipbone_b200.so (include/hipbone_b200.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels.  torch is used for device memory and streams (tensor.data_ptr(),
torch.cuda.current_stream().cuda_stream).  There is no CPU fallback: if the shared
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libhipbone_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the hipBone hot path)")

_lib = C.CDLL(LIB_PATH)

HB_OK = 0
ERRORS = {-1: "HB_ERR_ARG", -2: "HB_ERR_CONFIG", -3: "HB_ERR_GEOMETRY", -4: "HB_ERR_SETUP",
          -5: "HB_ERR_STATE", -6: "HB_ERR_BREAKDOWN", -7: "HB_ERR_CUDA", -8: "HB_ERR_NCCL",
          -9: "HB_ERR_OOM"}


class HBError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class hb_box(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("N", C.c_int32),
                ("ext", C.c_double * 3), ("mass_mode", C.c_int32)]


class hb_sizes(C.Structure):
    _fields_ = [("E_global", C.c_int64), ("E_local", C.c_int64), ("N_L", C.c_int64), ("N_G", C.c_int64),
                ("n_owned", C.c_int64), ("n_halo", C.c_int64), ("n_intA", C.c_int64),
                ("n_halo_elems", C.c_int64), ("n_intB", C.c_int64), ("n_neighbors", C.c_int32),
                ("rank", C.c_int32), ("P", C.c_int32), ("grid", C.c_int32 * 3)]


class hb_cg_result(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("rr0", C.c_double), ("rr_final", C.c_double)]


_p = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)

_SIGS = {
    "hb_last_error": (C.c_char_p, []),
    "hb_version": (C.c_int, []),
    "hb_gll": (C.c_int, [C.c_int, _dp, _dp, _dp]),
    "hb_rank_grid": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _i32p]),
    "hb_mesh_create": (C.c_int, [C.POINTER(hb_box), C.c_int, C.c_int, _i32p, C.c_uint64, C.POINTER(_p)]),
    "hb_mesh_sizes": (C.c_int, [_p, C.POINTER(hb_sizes)]),
    "hb_mesh_elements": (C.c_int, [_p, _i64p]),
    "hb_mesh_l2g": (C.c_int, [_p, _i64p]),
    "hb_mesh_local_index": (C.c_int, [_p, _i32p]),
    "hb_mesh_owned": (C.c_int, [_p, _i64p]),
    "hb_mesh_halo": (C.c_int, [_p, _i64p]),
    "hb_mesh_neighbors": (C.c_int, [_p, _i32p, _i64p, _i64p]),
    "hb_mesh_send_list": (C.c_int, [_p, C.c_int, _i64p]),
    "hb_mesh_geometry": (C.c_int, [_p, _dp]),
    "hb_mesh_set_geometry": (C.c_int, [_p, _dp]),
    "hb_mesh_mass": (C.c_int, [_p, _dp]),
    "hb_mesh_set_mass": (C.c_int, [_p, _dp]),
    "hb_mesh_destroy": (C.c_int, [_p]),
    "hb_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "hb_comm_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(_p)]),
    "hb_comm_destroy": (C.c_int, [_p]),
    "hb_comm_create_ipc": (C.c_int, [C.c_int, C.c_int, C.POINTER(_p)]),
    "hb_op_ipc_blob_size": (C.c_int, [_p, _i64p]),
    "hb_op_ipc_export": (C.c_int, [_p, C.POINTER(C.c_uint8)]),
    "hb_op_ipc_connect": (C.c_int, [_p, C.POINTER(C.c_uint8)]),
    "hb_op_set_ipc_direct": (C.c_int, [_p, C.c_int]),
    "hb_op_create": (C.c_int, [_p, _p, C.c_double, _p, C.POINTER(_p)]),
    "hb_op_apply": (C.c_int, [_p, _p, _p, _p]),
    "hb_forcing": (C.c_int, [_p, C.c_uint64, _p, _p]),
    "hb_dot": (C.c_int, [_p, _p, _p, _dp, _p]),
    "hb_cg_solve": (C.c_int, [_p, _p, _p, C.c_int32, C.c_double, _dp, C.POINTER(hb_cg_result), _p]),
    "hb_cg_solve_scattered": (C.c_int, [_p, _p, _p, C.c_int32, C.c_double, _dp, C.POINTER(hb_cg_result), _p]),
    "hb_cg_solve_host": (C.c_int, [_p, _dp, _dp, C.c_int32, C.c_double, _dp, C.POINTER(hb_cg_result), _p]),
    "hb_op_set_profiling": (C.c_int, [_p, C.c_int]),
    "hb_op_set_jacobi": (C.c_int, [_p, C.c_int, _p]),
    "hb_op_set_variant": (C.c_int, [_p, C.c_int, _p]),
    "hb_op_set_tolerance_loop": (C.c_int, [_p, C.c_int]),
    "hb_op_launch_shape": (C.c_int, [_p, _i32p]),
    "hb_op_set_timing_mode": (C.c_int, [_p, C.c_int]),
    "hb_op_jacobi_diagonal": (C.c_int, [_p, _p, _p]),
    "hb_op_kernel_time": (C.c_int, [_p, _i64p, _dp]),
    "hb_op_launch_count": (C.c_int, [_p, _i64p]),
    "hb_op_phase_times": (C.c_int, [_p, _dp]),
    "hb_op_sizes": (C.c_int, [_p, C.POINTER(hb_sizes)]),
    "hb_op_destroy": (C.c_int, [_p]),
    "hb_group_create": (C.c_int, [C.POINTER(_p), C.c_int, C.POINTER(_p)]),
    "hb_group_apply": (C.c_int, [_p, C.POINTER(_p), C.POINTER(_p), _p]),
    "hb_group_cg_solve": (C.c_int, [_p, C.POINTER(_p), C.POINTER(_p), C.c_int32, C.c_double, _dp,
                                    C.POINTER(hb_cg_result), _p]),
    "hb_group_destroy": (C.c_int, [_p]),
    "hb_stream_bench": (C.c_int, [C.c_int64, C.c_int, _dp]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def _check(code: int):
    if code != HB_OK:
        raise HBError(code, _lib.hb_last_error().decode(errors="replace"))


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _dev(t) -> int:
    """device pointer of a contiguous float64 CUDA tensor (or None -> NULL)"""
    if t is None:
        return None
    if not (t.is_cuda and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def version() -> int:
    return _lib.hb_version()


def gll(N: int):
    x = np.zeros(N + 1)
    w = np.zeros(N + 1)
    D = np.zeros((N + 1) * (N + 1))
    _check(_lib.hb_gll(N, _ptr(x, C.c_double), _ptr(w, C.c_double), _ptr(D, C.c_double)))
    return x, w, D.reshape(N + 1, N + 1)


def rank_grid(P: int, nx: int, ny: int, nz: int):
    g = np.zeros(3, dtype=np.int32)
    _check(_lib.hb_rank_grid(P, nx, ny, nz, _ptr(g, C.c_int32)))
    return tuple(int(v) for v in g)


def stream_bench(n_out: int, reps: int = 20) -> float:
    v = C.c_double()
    _check(_lib.hb_stream_bench(n_out, reps, C.byref(v)))
    return v.value


class Mesh:
    """Host-side box mesh / partition of one rank (hb_mesh_*)."""

    def __init__(self, nx, ny, nz, N, ext=(2.0, 2.0, 2.0), mass_mode=0, P=1, rank=0, grid=None, seed=0):
        box = hb_box(nx, ny, nz, N, (C.c_double * 3)(*ext), mass_mode)
        h = _p()
        g = None
        if grid is not None:
            self._grid = np.array(grid, dtype=np.int32)
            g = _ptr(self._grid, C.c_int32)
        _check(_lib.hb_mesh_create(C.byref(box), P, rank, g, seed, C.byref(h)))
        self._h = h
        self.N = N
        self.NP3 = (N + 1) ** 3
        s = hb_sizes()
        _check(_lib.hb_mesh_sizes(h, C.byref(s)))
        self.sizes = {f: (tuple(getattr(s, f)) if f == "grid" else getattr(s, f)) for f, _ in hb_sizes._fields_}

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.hb_mesh_destroy(self._h)
            self._h = None

    def _arr(self, fn, n, dtype, ctype, shape=None):
        a = np.zeros(n, dtype=dtype)
        _check(fn(self._h, _ptr(a, ctype)))
        return a.reshape(shape) if shape else a

    def elements(self):
        return self._arr(_lib.hb_mesh_elements, self.sizes["E_local"], np.int64, C.c_int64)

    def l2g(self):
        return self._arr(_lib.hb_mesh_l2g, self.sizes["N_L"], np.int64, C.c_int64, (-1, self.NP3))

    def local_index(self):
        return self._arr(_lib.hb_mesh_local_index, self.sizes["N_L"], np.int32, C.c_int32, (-1, self.NP3))

    def owned(self):
        return self._arr(_lib.hb_mesh_owned, self.sizes["n_owned"], np.int64, C.c_int64)

    def halo(self):
        return self._arr(_lib.hb_mesh_halo, self.sizes["n_halo"], np.int64, C.c_int64)

    def neighbors(self):
        n = self.sizes["n_neighbors"]
        r = np.zeros(n, dtype=np.int32)
        sc = np.zeros(n, dtype=np.int64)
        rc = np.zeros(n, dtype=np.int64)
        _check(_lib.hb_mesh_neighbors(self._h, _ptr(r, C.c_int32), _ptr(sc, C.c_int64), _ptr(rc, C.c_int64)))
        return r, sc, rc

    def send_list(self, q: int):
        _, sc, _ = self.neighbors()
        a = np.zeros(int(sc[q]), dtype=np.int64)
        _check(_lib.hb_mesh_send_list(self._h, q, _ptr(a, C.c_int64)))
        return a

    def geometry(self):
        return self._arr(_lib.hb_mesh_geometry, self.sizes["N_L"] * 6, np.float64, C.c_double, (-1, self.NP3, 6))

    def set_geometry(self, G: np.ndarray):
        G = np.ascontiguousarray(G, dtype=np.float64)
        if G.size != self.sizes["N_L"] * 6:
            raise ValueError("geometry must be [E_local][(N+1)^3][6]")
        _check(_lib.hb_mesh_set_geometry(self._h, _ptr(G, C.c_double)))

    def mass(self):
        return self._arr(_lib.hb_mesh_mass, self.sizes["N_L"], np.float64, C.c_double, (-1, self.NP3))

    def set_mass(self, M: np.ndarray):
        M = np.ascontiguousarray(M, dtype=np.float64)
        if M.size != self.sizes["N_L"]:
            raise ValueError("mass must be [E_local][(N+1)^3]")
        _check(_lib.hb_mesh_set_mass(self._h, _ptr(M, C.c_double)))


def comm_unique_id() -> bytes:
    a = (C.c_uint8 * 128)()
    _check(_lib.hb_comm_unique_id(a))
    return bytes(a)


class Comm:
    """Communicator of one rank: NCCL (`Comm(P, rank, uid)`, one GPU per rank) or the IPC
    peer-memory transport (`Comm.ipc(P, rank)`; ops on it need `Operator.ipc_connect`)."""

    def __init__(self, P: int, rank: int, uid: bytes | None = None, *, ipc: bool = False):
        h = _p()
        if ipc:
            _check(_lib.hb_comm_create_ipc(P, rank, C.byref(h)))
        else:
            a = (C.c_uint8 * 128).from_buffer_copy(uid)
            _check(_lib.hb_comm_create(P, rank, a, C.byref(h)))
        self._h = h
        self.ipc = ipc

    @classmethod
    def create_ipc(cls, P: int, rank: int) -> "Comm":
        return cls(P, rank, ipc=True)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.hb_comm_destroy(self._h)
            self._h = None


class Operator:
    """Device operator of one rank (hb_op_*).  Vectors are float64 CUDA tensors of length n_owned."""

    def __init__(self, mesh: Mesh, lam: float = 1.0, comm: Comm | None = None, stream=None):
        h = _p()
        _check(_lib.hb_op_create(mesh._h, comm._h if comm else None, lam, _stream(stream), C.byref(h)))
        self._h = h
        self.mesh = mesh
        self.comm = comm
        self.lam = lam
        s = hb_sizes()
        _check(_lib.hb_op_sizes(h, C.byref(s)))
        self.n_owned = s.n_owned

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.hb_op_destroy(self._h)
            self._h = None

    def ipc_export(self) -> bytes:
        """This rank's IPC export record (hb_op_ipc_export)."""
        n = C.c_int64()
        _check(_lib.hb_op_ipc_blob_size(self._h, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _check(_lib.hb_op_ipc_export(self._h, buf))
        return bytes(buf)

    def ipc_connect(self, records) -> None:
        """Map the peers' buffers from the all-gathered records (rank order; hb_op_ipc_connect)."""
        blob = b"".join(records)
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(_lib.hb_op_ipc_connect(self._h, buf))

    def set_ipc_direct(self, enable: bool) -> None:
        """IPC transport, CG: halo elements read / add into the owners' vectors directly (default)."""
        _check(_lib.hb_op_set_ipc_direct(self._h, int(bool(enable))))

    def apply(self, x, y, stream=None):
        _check(_lib.hb_op_apply(self._h, _dev(x), _dev(y), _stream(stream)))

    def forcing(self, seed: int, b, stream=None):
        _check(_lib.hb_forcing(self._h, seed, _dev(b), _stream(stream)))

    def dot(self, a, b, stream=None) -> float:
        v = C.c_double()
        _check(_lib.hb_dot(self._h, _dev(a), _dev(b), C.byref(v), _stream(stream)))
        return v.value

    def cg(self, b, x, max_iters: int, eps: float = -1.0, stream=None):
        """Returns (iterations, rr history np.array[iterations+1])."""
        hist = np.zeros(max_iters + 1)
        res = hb_cg_result()
        _check(_lib.hb_cg_solve(self._h, _dev(b), _dev(x), max_iters, eps, _ptr(hist, C.c_double),
                                C.byref(res), _stream(stream)))
        return res.iterations, hist[:res.iterations + 1].copy()

    def cg_scattered(self, b, x, max_iters: int, eps: float = -1.0, stream=None):
        """NekBone's scattered-storage CG (P = 1, mass mode 0); same return as cg()."""
        hist = np.zeros(max_iters + 1)
        res = hb_cg_result()
        _check(_lib.hb_cg_solve_scattered(self._h, _dev(b), _dev(x), max_iters, eps, _ptr(hist, C.c_double),
                                          C.byref(res), _stream(stream)))
        return res.iterations, hist[:res.iterations + 1].copy()

    def cg_host(self, b: np.ndarray, x: np.ndarray, max_iters: int, eps: float = -1.0, stream=None,
                hist: bool = True):
        """CG on host buffers (copies inside the call); x is written in place."""
        assert b.dtype == np.float64 and x.dtype == np.float64 and b.flags.c_contiguous and x.flags.c_contiguous
        h = np.zeros(max_iters + 1) if hist else None
        res = hb_cg_result()
        _check(_lib.hb_cg_solve_host(self._h, _ptr(b, C.c_double), _ptr(x, C.c_double), max_iters, eps,
                                     _ptr(h, C.c_double) if hist else None, C.byref(res), _stream(stream)))
        return res.iterations, (h[:res.iterations + 1].copy() if hist else None)

    def set_variant(self, variant: int, stream=None):
        """0: fused scatter-add (default); 1: y_L + deterministic CSR gather (P = 1)."""
        _check(_lib.hb_op_set_variant(self._h, int(variant), _stream(stream)))

    def set_tolerance_loop(self, device: bool):
        """Tolerance-mode CG loop: on the device (one graph, WHILE node; default) or host-driven."""
        _check(_lib.hb_op_set_tolerance_loop(self._h, int(bool(device))))

    def set_timing_mode(self, vec_only: bool):
        """Measurement hook: fixed-mode CG without the operator launches (vector kernels only)."""
        _check(_lib.hb_op_set_timing_mode(self._h, int(bool(vec_only))))

    def launch_shape(self) -> dict:
        """Operator launch shape: resident grid, threads per CTA, elements per CTA, shared bytes."""
        a = np.zeros(4, dtype=np.int32)
        _check(_lib.hb_op_launch_shape(self._h, _ptr(a, C.c_int32)))
        return {"grid": int(a[0]), "block": int(a[1]), "epb": int(a[2]), "smem": int(a[3])}

    def set_jacobi(self, enable: bool, stream=None):
        """Jacobi-preconditioned CG for subsequent cg() calls (P = 1)."""
        _check(_lib.hb_op_set_jacobi(self._h, int(bool(enable)), _stream(stream)))

    def jacobi_diagonal(self, out, stream=None):
        """diag(A) on owned DOFs into the CUDA tensor `out` (after set_jacobi(True))."""
        _check(_lib.hb_op_jacobi_diagonal(self._h, _dev(out), _stream(stream)))

    def set_profiling(self, enable, stride: int = 1):
        """enable=False: off; else time every `stride`-th operator launch with CUDA events."""
        _check(_lib.hb_op_set_profiling(self._h, int(stride) if enable else 0))

    def kernel_time(self):
        n = C.c_int64()
        t = C.c_double()
        _check(_lib.hb_op_kernel_time(self._h, C.byref(n), C.byref(t)))
        return n.value, t.value

    def phase_times(self):
        """(operator, x/r update, p update) mean seconds of the timed CG iterations."""
        a = np.zeros(3)
        _check(_lib.hb_op_phase_times(self._h, _ptr(a, C.c_double)))
        return tuple(float(v) for v in a)

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(_lib.hb_op_launch_count(self._h, C.byref(n)))
        return n.value


class Group:
    """Loopback group: P comm-less ops of one partition driven in one process on one GPU."""

    def __init__(self, ops: list[Operator]):
        arr = (_p * len(ops))(*[o._h for o in ops])
        h = _p()
        _check(_lib.hb_group_create(arr, len(ops), C.byref(h)))
        self._h = h
        self.ops = ops

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.hb_group_destroy(self._h)
            self._h = None

    @staticmethod
    def _ptrs(ts):
        return (_p * len(ts))(*[_dev(t) for t in ts])

    def apply(self, xs, ys, stream=None):
        _check(_lib.hb_group_apply(self._h, self._ptrs(xs), self._ptrs(ys), _stream(stream)))

    def cg(self, bs, xs, max_iters: int, eps: float = -1.0, stream=None):
        hist = np.zeros(max_iters + 1)
        res = hb_cg_result()
        _check(_lib.hb_group_cg_solve(self._h, self._ptrs(bs), self._ptrs(xs), max_iters, eps,
                                      _ptr(hist, C.c_double), C.byref(res), _stream(stream)))
        return res.iterations, hist[:res.iterations + 1].copy()
