"""Thin Python binding of include/mf.h (ctypes).  Argument marshalling only:
every step of the hot path runs in libmf_b200.so's CUDA kernels; PyTorch
supplies device memory, the current CUDA stream and the process group that
broadcasts the NCCL id.  There is no CPU fallback: if the library or a CUDA
device is missing, constructing an Operator raises."""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

MF_OK = 0
STATUS = {
    -1: "MF_ERR_ARGUMENT", -2: "MF_ERR_LENGTH", -3: "MF_ERR_SINGULAR", -4: "MF_ERR_MAX_ITERATIONS",
    -5: "MF_ERR_BREAKDOWN", -6: "MF_ERR_CUDA", -7: "MF_ERR_NCCL", -8: "MF_ERR_OUT_OF_MEMORY",
}
GEOM = {"cartesian": 0, "sine": 1}
VARIANT = {"auto": 0, "general": 1, "plane": 3, "halo": 6}


class MFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class Mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_cells", ctypes.c_int64 * 3), ("lower", ctypes.c_double * 3),
                ("upper", ctypes.c_double * 3), ("geometry", ctypes.c_int32), ("deform_eps", ctypes.c_double),
                ("dirichlet_faces", ctypes.c_uint32)]


class Coeff(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("value", ctypes.c_double)]


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world_size", ctypes.c_int32),
                ("nccl_unique_id", ctypes.POINTER(ctypes.c_uint8)), ("device", ctypes.c_int32)]


class CGParams(ctypes.Structure):
    _fields_ = [("rel_tol", ctypes.c_double), ("max_iter", ctypes.c_int32), ("cheb_degree", ctypes.c_int32),
                ("cheb_range", ctypes.c_double), ("cheb_safety", ctypes.c_double), ("eig_cg_steps", ctypes.c_int32),
                ("precision", ctypes.c_int32)]


class CGResultC(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("final_rel_residual", ctypes.c_double),
                ("lambda_max", ctypes.c_double)]


class MGParams(ctypes.Structure):
    _fields_ = [("n_levels", ctypes.c_int32), ("max_coarse_dofs", ctypes.c_int64), ("smooth_degree", ctypes.c_int32),
                ("smooth_range", ctypes.c_double), ("smooth_safety", ctypes.c_double), ("eig_cg_steps", ctypes.c_int32),
                ("precision", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("degree", ctypes.c_int32), ("geometry", ctypes.c_int32),
                ("coeff_kind", ctypes.c_int32), ("apply_variant", ctypes.c_int32),
                ("n_cells_local", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("bytes_algorithmic", ctypes.c_int64), ("flops_algorithmic", ctypes.c_double)]


class HexMeshC(ctypes.Structure):
    _fields_ = [("n_vertices", ctypes.c_int64), ("n_cells", ctypes.c_int64), ("n_dofs", ctypes.c_int64),
                ("n_lines", ctypes.c_int64), ("n_dirichlet", ctypes.c_int64),
                ("vertices", ctypes.c_void_p), ("cell_vertices", ctypes.c_void_p), ("cell_dofs", ctypes.c_void_p),
                ("line_ptr", ctypes.c_void_p), ("line_dof", ctypes.c_void_p), ("line_w", ctypes.c_void_p),
                ("dirichlet_dofs", ctypes.c_void_p)]


EXPORTS = ["mf_create", "mf_destroy", "mf_last_error", "mf_nccl_unique_id", "mf_sizes", "mf_set_stream",
           "mf_apply", "mf_apply_host", "mf_diagonal", "mf_estimate_lambda_max", "mf_chebyshev",
           "mf_cg_solve", "mf_get_info", "mf_set_apply_variant", "mf_set_kernel_timing", "mf_kernel_timing",
           "mf_partition", "mf_mg_create", "mf_mg_destroy", "mf_mg_levels", "mf_mg_level_size", "mf_mg_level_op",
           "mf_mg_level_lambda", "mf_mg_prolongate", "mf_mg_restrict", "mf_mg_vcycle", "mf_mg_cg_solve",
           "mf_mg_set_stream", "mf_apply_f32", "mf_create_dg", "mf_hng_create", "mf_hng_destroy", "mf_hng_sizes",
           "mf_hng_apply", "mf_hng_set_stream", "mf_create_hex", "mf_hex_number_dofs", "mf_apply_split_part",
           "mf_sync"]

_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libmf_b200.so (built in-tree by build.py).  Loading needs no GPU."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MF_LIB_PATH") or _build.LIB  # (MF_LIB_PATH: kernel experiments)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `python -m paper_1910_13247_b200.build` (no CPU fallback)")
    L = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    dp = ctypes.POINTER(ctypes.c_double)
    i64 = ctypes.c_int64
    i64p = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "mf_create": [ctypes.POINTER(Mesh), ctypes.c_int32, ctypes.POINTER(Coeff), ctypes.POINTER(Dist),
                      ctypes.POINTER(vp)],
        "mf_sizes": [vp, i64p, i64p, i64p, i64p],
        "mf_set_stream": [vp, vp],
        "mf_apply": [vp, vp, i64, vp, i64],
        "mf_apply_host": [vp, dp, i64, dp, i64],
        "mf_diagonal": [vp, vp, i64],
        "mf_estimate_lambda_max": [vp, ctypes.c_int32, dp],
        "mf_chebyshev": [vp, vp, vp, i64, ctypes.c_double, ctypes.c_int32, ctypes.c_double],
        "mf_cg_solve": [vp, vp, vp, i64, ctypes.POINTER(CGParams), ctypes.POINTER(CGResultC), dp, ctypes.c_int32],
        "mf_get_info": [vp, ctypes.POINTER(Info)],
        "mf_set_apply_variant": [vp, ctypes.c_int32],
        "mf_set_kernel_timing": [vp, ctypes.c_int32],
        "mf_kernel_timing": [vp, dp, i64p],
        "mf_nccl_unique_id": [ctypes.POINTER(ctypes.c_uint8)],
        "mf_partition": [ctypes.POINTER(Mesh), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                         i64p, i64p, i64p, i64p, i64p, i64p],
        "mf_mg_create": [ctypes.POINTER(Mesh), ctypes.c_int32, ctypes.POINTER(Coeff), ctypes.POINTER(MGParams),
                         ctypes.POINTER(vp)],
        "mf_mg_levels": [vp, ctypes.POINTER(ctypes.c_int32)],
        "mf_mg_level_size": [vp, ctypes.c_int32, i64p],
        "mf_mg_level_op": [vp, ctypes.c_int32, ctypes.POINTER(vp)],
        "mf_mg_level_lambda": [vp, ctypes.c_int32, dp],
        "mf_mg_prolongate": [vp, ctypes.c_int32, vp, vp],
        "mf_mg_restrict": [vp, ctypes.c_int32, vp, vp],
        "mf_mg_vcycle": [vp, vp, vp, i64],
        "mf_mg_cg_solve": [vp, vp, vp, i64, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(CGResultC), dp,
                           ctypes.c_int32],
        "mf_mg_set_stream": [vp, vp],
        "mf_apply_f32": [vp, vp, i64, vp, i64],
        "mf_apply_split_part": [vp, vp, i64, vp, i64, ctypes.c_int32],
        "mf_sync": [vp],
        "mf_create_dg": [ctypes.POINTER(Mesh), ctypes.c_int32, ctypes.POINTER(Coeff), ctypes.POINTER(vp)],
        "mf_hng_create": [dp, dp, ctypes.c_double, i64p, i64, ctypes.c_int32, ctypes.POINTER(Coeff),
                          ctypes.POINTER(vp)],
        "mf_hng_sizes": [vp, i64p, i64p],
        "mf_hng_apply": [vp, vp, i64, vp, i64],
        "mf_hng_set_stream": [vp, vp],
        "mf_create_hex": [ctypes.POINTER(HexMeshC), ctypes.c_int32, ctypes.POINTER(Coeff), ctypes.POINTER(vp)],
        "mf_hex_number_dofs": [ctypes.c_int32, i64, vp, vp, i64p, vp, i64],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.mf_destroy.argtypes = [vp]
    L.mf_destroy.restype = None
    L.mf_mg_destroy.argtypes = [vp]
    L.mf_mg_destroy.restype = None
    L.mf_hng_destroy.argtypes = [vp]
    L.mf_hng_destroy.restype = None
    L.mf_last_error.argtypes = []
    L.mf_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(code: int):
    if code != MF_OK:
        raise MFError(code, load().mf_last_error().decode())


def make_mesh(n_cells, dim=None, lower=None, upper=None, geometry="cartesian", eps=0.1, dirichlet_faces=None):
    dim = dim or len(n_cells)
    m = Mesh()
    m.dim = dim
    for e in range(3):
        m.n_cells[e] = int(n_cells[e]) if e < dim else 1
        m.lower[e] = float(lower[e]) if lower is not None and e < dim else 0.0
        m.upper[e] = float(upper[e]) if upper is not None and e < dim else 1.0
    m.geometry = GEOM[geometry] if isinstance(geometry, str) else int(geometry)
    m.deform_eps = eps
    m.dirichlet_faces = ((1 << (2 * dim)) - 1) if dirichlet_faces is None else int(dirichlet_faces)
    return m


def partition(n_cells, degree, rank, world_size, **mesh_kw) -> dict:
    """mf_partition: the z-slab of `rank` (host arithmetic only, no GPU needed)."""
    m = make_mesh(n_cells, **mesh_kw)
    vals = [ctypes.c_int64() for _ in range(6)]
    _check(load().mf_partition(ctypes.byref(m), degree, rank, world_size, *[ctypes.byref(v) for v in vals]))
    keys = ["cz0", "cz1", "first_global", "n_local", "n_owned", "plane"]
    return {k: v.value for k, v in zip(keys, vals)}


@dataclass
class CGResult:
    iterations: int
    final_rel_residual: float
    lambda_max: float
    history: np.ndarray


class Operator:
    """v = A u for the Q_k Laplacian on a brick (see include/mf.h).

    Vectors are torch.float64 CUDA tensors of length n_local (the rank's slice
    [first_global, first_global + n_local) of the x-fastest global vector)."""

    def __init__(self, n_cells, degree, dim=None, lower=None, upper=None, geometry="cartesian", eps=0.1,
                 coeff=1.0, dirichlet_faces=None, group=None, device=None, discretization="cg", slab=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1910_13247_b200 needs a CUDA device (no CPU fallback)")
        self._torch = torch
        L = load()
        dim = dim or len(n_cells)
        m = Mesh()
        m.dim = dim
        for e in range(3):
            m.n_cells[e] = int(n_cells[e]) if e < dim else 1
            m.lower[e] = float(lower[e]) if lower is not None and e < dim else 0.0
            m.upper[e] = float(upper[e]) if upper is not None and e < dim else 1.0
        m.geometry = GEOM[geometry] if isinstance(geometry, str) else int(geometry)
        m.deform_eps = eps
        m.dirichlet_faces = ((1 << (2 * dim)) - 1) if dirichlet_faces is None else int(dirichlet_faces)
        c = Coeff()
        if isinstance(coeff, str):
            assert coeff == "variable"
            c.kind, c.value = 1, 0.0
        else:
            c.kind, c.value = 0, float(coeff)
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        dist = Dist()
        dist.device = device
        self._uid = None
        if group is not None and torch.distributed.get_world_size(group) > 1:
            import torch.distributed as tdist

            rank, world = tdist.get_rank(group), tdist.get_world_size(group)
            obj = [None]
            if rank == 0:
                buf = (ctypes.c_uint8 * 128)()
                _check(L.mf_nccl_unique_id(buf))
                obj = [bytes(buf)]
            tdist.broadcast_object_list(obj, src=tdist.get_global_rank(group, 0), group=group)
            self._uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
            dist.rank, dist.world_size = rank, world
            dist.nccl_unique_id = ctypes.cast(self._uid, ctypes.POINTER(ctypes.c_uint8))
        elif slab is not None:  # detached slab (rank, world): partial sums on shared planes, no NCCL
            dist.rank, dist.world_size = int(slab[0]), int(slab[1])
        else:
            dist.rank, dist.world_size = 0, 1
        with torch.cuda.device(device):
            h = ctypes.c_void_p()
            if discretization == "dg":  # symmetric interior penalty DG (mf_create_dg)
                _check(L.mf_create_dg(ctypes.byref(m), degree, ctypes.byref(c), ctypes.byref(h)))
            else:
                _check(L.mf_create(ctypes.byref(m), degree, ctypes.byref(c), ctypes.byref(dist), ctypes.byref(h)))
        self._h = h
        self.dim, self.degree, self.mesh = dim, degree, m
        a, b, cc, d = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(L.mf_sizes(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(cc), ctypes.byref(d)))
        self.n_local, self.first_global, self.n_global, self.n_owned = a.value, b.value, cc.value, d.value

    def close(self):
        if getattr(self, "_h", None):
            load().mf_destroy(self._h)
            self._h = None

    __del__ = close

    # -- helpers -------------------------------------------------------------
    def _stream(self):
        _check(load().mf_set_stream(self._h, ctypes.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)))

    def _vec(self, x, name):
        t = self._torch
        if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float64 and x.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
        if x.device != self.device:
            raise TypeError(f"{name} is on {x.device}, the operator on {self.device}")
        return ctypes.c_void_p(x.data_ptr())

    def new_vector(self):
        return self._torch.zeros(self.n_local, dtype=self._torch.float64, device=self.device)

    # -- C-ABI calls ---------------------------------------------------------
    def apply(self, src, dst=None):
        dst = self.new_vector() if dst is None else dst
        self._stream()
        _check(load().mf_apply(self._h, self._vec(src, "src"), src.numel(), self._vec(dst, "dst"), dst.numel()))
        return dst

    def apply_split_part(self, src, dst, part: int):
        """One part of the overlapped multi-GPU launch sequence on this GPU (mf_apply_split_part:
        1 = the cell layers next to the shared z-planes, 2 = the interior layers)."""
        self._stream()
        _check(load().mf_apply_split_part(self._h, self._vec(src, "src"), src.numel(), self._vec(dst, "dst"),
                                          dst.numel(), int(part)))
        return dst

    def sync(self):
        """mf_sync: wait for the op's stream (watching the communicator on N > 1)."""
        _check(load().mf_sync(self._h))

    def apply_f32(self, src, dst=None):
        """The FP32 instance of the apply (mixed-precision multigrid); float32 CUDA tensors."""
        t = self._torch
        dst = t.zeros(self.n_local, dtype=t.float32, device=self.device) if dst is None else dst
        for x, name in ((src, "src"), (dst, "dst")):
            if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float32 and x.is_contiguous()):
                raise TypeError(f"{name} must be a contiguous float32 CUDA tensor")
        self._stream()
        _check(load().mf_apply_f32(self._h, ctypes.c_void_p(src.data_ptr()), src.numel(),
                                   ctypes.c_void_p(dst.data_ptr()), dst.numel()))
        return dst

    def apply_host(self, src: np.ndarray, dst: np.ndarray | None = None) -> np.ndarray:
        src = np.ascontiguousarray(src, dtype=np.float64)
        if dst is None:
            dst = np.empty_like(src)
        elif not (isinstance(dst, np.ndarray) and dst.dtype == np.float64 and dst.flags["C_CONTIGUOUS"]
                  and dst.flags["WRITEABLE"] and dst.size == self.n_local):
            # the C side writes n_local doubles through dst's data pointer
            raise TypeError(f"dst must be a writeable C-contiguous float64 array of {self.n_local} entries")
        dp = ctypes.POINTER(ctypes.c_double)
        self._stream()
        _check(load().mf_apply_host(self._h, src.ctypes.data_as(dp), src.size, dst.ctypes.data_as(dp), dst.size))
        return dst

    def apply_host_ptr(self, src_ptr: int, dst_ptr: int):
        """mf_apply_host on raw host pointers (e.g. pinned torch tensors)."""
        dp = ctypes.POINTER(ctypes.c_double)
        self._stream()
        _check(load().mf_apply_host(self._h, ctypes.cast(src_ptr, dp), self.n_local, ctypes.cast(dst_ptr, dp),
                                    self.n_local))

    def diagonal(self, out=None):
        out = self.new_vector() if out is None else out
        self._stream()
        _check(load().mf_diagonal(self._h, self._vec(out, "diag"), out.numel()))
        return out

    def estimate_lambda_max(self, steps: int = 12) -> float:
        lam = ctypes.c_double()
        self._stream()
        _check(load().mf_estimate_lambda_max(self._h, steps, ctypes.byref(lam)))
        return lam.value

    def chebyshev(self, r, lam: float, degree: int = 6, smoothing_range: float = 20.0, out=None):
        out = self.new_vector() if out is None else out
        self._stream()
        _check(load().mf_chebyshev(self._h, self._vec(r, "r"), self._vec(out, "z"), r.numel(), lam, degree,
                                   smoothing_range))
        return out

    def cg_solve(self, b, x=None, rel_tol=1e-10, max_iter=10000, cheb_degree=6, cheb_range=20.0,
                 cheb_safety=1.2, eig_cg_steps=12, history_cap=20000, precision="fp64"):
        """Chebyshev-Jacobi PCG; precision="mixed" runs the Chebyshev preconditioner in FP32."""
        x = self.new_vector() if x is None else x
        p = CGParams(rel_tol, max_iter, cheb_degree, cheb_range, cheb_safety, eig_cg_steps,
                     {"fp64": 0, "mixed": 1}[precision])
        r = CGResultC()
        hist = np.zeros(history_cap)
        self._stream()
        code = load().mf_cg_solve(self._h, self._vec(b, "b"), self._vec(x, "x"), b.numel(), ctypes.byref(p),
                                  ctypes.byref(r), hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), history_cap)
        _check(code)
        return x, CGResult(r.iterations, r.final_rel_residual, r.lambda_max, hist[:r.iterations].copy())

    def info(self) -> dict:
        i = Info()
        _check(load().mf_get_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in Info._fields_}

    def set_variant(self, variant):
        v = VARIANT[variant] if isinstance(variant, str) else int(variant)
        _check(load().mf_set_apply_variant(self._h, v))

    def kernel_timing(self, enable: bool):
        _check(load().mf_set_kernel_timing(self._h, 1 if enable else 0))

    def kernel_time(self):
        """(summed ms, launches) of the dominant apply kernel since kernel_timing(True)."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _check(load().mf_kernel_timing(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value


def hex_number_dofs(cell_vertices: np.ndarray, degree: int):
    """mf_hex_number_dofs (host only): DoF numbering of a conforming hex mesh.
    Returns (cell_dofs [n_cells][(k+1)^3] int32, n_dofs, is_boundary [n_dofs] bool)."""
    cv = np.ascontiguousarray(cell_vertices, dtype=np.int32)
    nc = cv.shape[0]
    cd = np.empty((nc, (degree + 1) ** 3), dtype=np.int32)
    cap = cd.size + 1
    bnd = np.empty(cap, dtype=np.uint8)
    n = ctypes.c_int64()
    _check(load().mf_hex_number_dofs(degree, nc, cv.ctypes.data, cd.ctypes.data, ctypes.byref(n),
                                     bnd.ctypes.data, cap))
    return cd, n.value, bnd[:n.value].astype(bool)


class HexOperator(Operator):
    """v = A u for continuous Q_k on a general unstructured hex mesh (mf_create_hex;
    include/mf.h): trilinear cells, cell_dofs (>= 0 DoF, < 0 constraint line -1 - v),
    constraint lines as (dof, weight) lists, Dirichlet DoFs with identity rows.  All
    Operator methods except the brick-only ones (apply_f32, set_variant) apply."""

    def __init__(self, vertices, cell_vertices, degree, cell_dofs, n_dofs, lines=(), dirichlet=(), coeff=1.0,
                 device=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1910_13247_b200 needs a CUDA device (no CPU fallback)")
        self._torch = torch
        L = load()
        V = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        CV = np.ascontiguousarray(cell_vertices, dtype=np.int32).reshape(-1, 8)
        CD = np.ascontiguousarray(cell_dofs, dtype=np.int32).reshape(CV.shape[0], -1)
        lp = np.zeros(len(lines) + 1, dtype=np.int32)
        for i, line in enumerate(lines):
            lp[i + 1] = lp[i] + len(line)
        ld = np.array([d for line in lines for d, _ in line] or [0], dtype=np.int32)
        lw = np.array([w for line in lines for _, w in line] or [0.0], dtype=np.float64)
        D = np.ascontiguousarray(np.asarray(dirichlet, dtype=np.int64).reshape(-1), dtype=np.int32)
        D = D if D.size else np.zeros(1, dtype=np.int32)
        m = HexMeshC()
        m.n_vertices, m.n_cells, m.n_dofs = V.shape[0], CV.shape[0], int(n_dofs)
        m.n_lines, m.n_dirichlet = len(lines), len(np.asarray(dirichlet).reshape(-1))
        m.vertices, m.cell_vertices, m.cell_dofs = V.ctypes.data, CV.ctypes.data, CD.ctypes.data
        m.line_ptr, m.line_dof, m.line_w, m.dirichlet_dofs = lp.ctypes.data, ld.ctypes.data, lw.ctypes.data, D.ctypes.data
        c = Coeff()
        if isinstance(coeff, str):
            assert coeff == "variable"
            c.kind, c.value = 1, 0.0
        else:
            c.kind, c.value = 0, float(coeff)
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self._uid = None
        with torch.cuda.device(device):
            h = ctypes.c_void_p()
            _check(L.mf_create_hex(ctypes.byref(m), degree, ctypes.byref(c), ctypes.byref(h)))
        self._h = h
        self.dim, self.degree, self.mesh = 3, degree, None
        self.n_local = self.n_global = self.n_owned = int(n_dofs)
        self.first_global = 0


class Multigrid:
    """Geometric multigrid on the globally refined brick (include/mf.h, mf_mg_*):
    level l = 0 (coarsest) .. n_levels - 1 (the given mesh); V-cycle with
    Chebyshev(smooth_degree) smoothing and a dense coarse solve; MG-preconditioned CG."""

    def __init__(self, n_cells, degree, lower=None, upper=None, geometry="cartesian", eps=0.1, coeff=1.0,
                 dirichlet_faces=None, n_levels=0, max_coarse_dofs=1000, smooth_degree=6, smooth_range=20.0,
                 smooth_safety=1.2, eig_cg_steps=12, precision="fp64"):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1910_13247_b200 needs a CUDA device (no CPU fallback)")
        self._torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())
        m = make_mesh(n_cells, 3, lower, upper, geometry, eps, dirichlet_faces)
        c = Coeff()
        c.kind, c.value = (1, 0.0) if coeff == "variable" else (0, float(coeff))
        prm = MGParams(n_levels, max_coarse_dofs, smooth_degree, smooth_range, smooth_safety, eig_cg_steps,
                       {"fp64": 0, "mixed": 1}[precision])
        h = ctypes.c_void_p()
        L = load()
        _check(L.mf_mg_create(ctypes.byref(m), degree, ctypes.byref(c), ctypes.byref(prm), ctypes.byref(h)))
        self._h = h
        nl = ctypes.c_int32()
        _check(L.mf_mg_levels(h, ctypes.byref(nl)))
        self.n_levels = nl.value
        self.sizes = []
        for l in range(self.n_levels):
            n = ctypes.c_int64()
            _check(L.mf_mg_level_size(h, l, ctypes.byref(n)))
            self.sizes.append(n.value)
        self.n_local = self.sizes[-1]

    def close(self):
        if getattr(self, "_h", None):
            load().mf_mg_destroy(self._h)
            self._h = None

    __del__ = close

    def _stream(self):
        _check(load().mf_mg_set_stream(self._h, ctypes.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)))

    def _vec(self, x, n, name):
        t = self._torch
        if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float64 and x.is_contiguous() and x.numel() == n):
            raise TypeError(f"{name} must be a contiguous float64 CUDA tensor of {n} entries")
        return ctypes.c_void_p(x.data_ptr())

    def new_vector(self, level=None):
        n = self.sizes[-1 if level is None else level]
        return self._torch.zeros(n, dtype=self._torch.float64, device=self.device)

    def level_lambda(self, level: int) -> float:
        v = ctypes.c_double()
        _check(load().mf_mg_level_lambda(self._h, level, ctypes.byref(v)))
        return v.value

    def level_apply(self, level: int, x, out=None):
        out = self.new_vector(level) if out is None else out
        op = ctypes.c_void_p()
        _check(load().mf_mg_level_op(self._h, level, ctypes.byref(op)))
        self._stream()
        n = self.sizes[level]
        _check(load().mf_apply(op, self._vec(x, n, "x"), n, self._vec(out, n, "out"), n))
        return out

    def prolongate(self, level: int, coarse, out=None):
        out = self.new_vector(level) if out is None else out
        self._stream()
        _check(load().mf_mg_prolongate(self._h, level, self._vec(coarse, self.sizes[level - 1], "coarse"),
                                       self._vec(out, self.sizes[level], "fine")))
        return out

    def restrict(self, level: int, fine, out=None):
        out = self.new_vector(level - 1) if out is None else out
        self._stream()
        _check(load().mf_mg_restrict(self._h, level, self._vec(fine, self.sizes[level], "fine"),
                                     self._vec(out, self.sizes[level - 1], "coarse")))
        return out

    def vcycle(self, b, out=None):
        out = self.new_vector() if out is None else out
        self._stream()
        _check(load().mf_mg_vcycle(self._h, self._vec(b, self.n_local, "b"), self._vec(out, self.n_local, "x"),
                                   self.n_local))
        return out

    def cg_solve(self, b, x=None, rel_tol=1e-10, max_iter=1000, history_cap=2000):
        x = self.new_vector() if x is None else x
        r = CGResultC()
        hist = np.zeros(history_cap)
        self._stream()
        _check(load().mf_mg_cg_solve(self._h, self._vec(b, self.n_local, "b"), self._vec(x, self.n_local, "x"),
                                     self.n_local, rel_tol, max_iter, ctypes.byref(r),
                                     hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), history_cap))
        return x, CGResult(r.iterations, r.final_rel_residual, r.lambda_max, hist[:r.iterations].copy())


class HangingNodeOperator:
    """Q_k Laplacian on the two-block mesh with one 2:1 interface at z = z_mid
    (include/mf.h, mf_hng_*): a coarse lower brick of n_cells_coarse cells and an upper
    brick refined once more, hanging interface nodes eliminated by interpolation."""

    def __init__(self, n_cells_coarse, nz_fine, degree, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0), z_mid=0.5,
                 coeff=1.0):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1910_13247_b200 needs a CUDA device (no CPU fallback)")
        self._torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())
        c = Coeff()
        c.kind, c.value = 0, float(coeff)
        lo = (ctypes.c_double * 3)(*lower)
        hi = (ctypes.c_double * 3)(*upper)
        nc = (ctypes.c_int64 * 3)(*n_cells_coarse)
        h = ctypes.c_void_p()
        L = load()
        _check(L.mf_hng_create(lo, hi, z_mid, nc, nz_fine, degree, ctypes.byref(c), ctypes.byref(h)))
        self._h = h
        n, nC = ctypes.c_int64(), ctypes.c_int64()
        _check(L.mf_hng_sizes(h, ctypes.byref(n), ctypes.byref(nC)))
        self.n_local, self.n_coarse = n.value, nC.value

    def close(self):
        if getattr(self, "_h", None):
            load().mf_hng_destroy(self._h)
            self._h = None

    __del__ = close

    def apply(self, src, dst=None):
        t = self._torch
        dst = t.zeros(self.n_local, dtype=t.float64, device=self.device) if dst is None else dst
        for x, name in ((src, "src"), (dst, "dst")):
            if not (isinstance(x, t.Tensor) and x.is_cuda and x.dtype == t.float64 and x.is_contiguous()
                    and x.numel() == self.n_local):
                raise TypeError(f"{name} must be a contiguous float64 CUDA tensor of {self.n_local} entries")
        _check(load().mf_hng_set_stream(self._h, ctypes.c_void_p(t.cuda.current_stream(self.device).cuda_stream)))
        _check(load().mf_hng_apply(self._h, ctypes.c_void_p(src.data_ptr()), self.n_local,
                                   ctypes.c_void_p(dst.data_ptr()), self.n_local))
        return dst
