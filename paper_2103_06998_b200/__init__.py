"""B200-native ADI isogeometric Maxwell time stepper (arXiv 2103.06998).

Thin ctypes binding over ``libadimaxwell.so`` (C ABI in ``include/adi_maxwell.h``):
argument marshalling only -- every step of the hot path runs in the library's
sm_100a CUDA kernels.  There is no CPU fallback: if the library or a CUDA
device is missing, the calls raise.

PyTorch is used for device memory (torch tensors may be passed as device
pointers) and nothing else.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
# ADI_LIB selects another build of the library (tuning experiments); default: the in-tree build
LIB_PATH = os.environ.get("ADI_LIB") or os.path.join(_HERE, "lib", "libadimaxwell.so")
CSRC = os.path.join(_HERE, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("adi_maxwell.cu", "degree.cu", "rhs.cuh", "dispatch.h", "setup_kernels.cuh", "sweep.cuh", "sweep_tw.cuh", "sweep_tma.cuh", "sweep_res.cuh", "rhs3.cuh")] + [
    os.path.join(_ROOT, "include", "adi_maxwell.h")]
DEGREES = (1, 2, 3, 4, 5)
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC"]

ADI_OK, ADI_ERR_ARG, ADI_ERR_STATE, ADI_ERR_SINGULAR, ADI_ERR_CUDA, ADI_ERR_NCCL, ADI_ERR_OOM = range(7)
ADI_BC_PEC, ADI_BC_NATURAL = 0, 1
K_CLASSES = ["rhs_e", "rhs_h", "sweep_mass", "sweep_mod", "other", "sweep_der"]

EXPORTS = [
    "adi_create", "adi_destroy", "adi_layout", "adi_set_tau", "adi_set_materials", "adi_set_materials_tf",
    "adi_set_fields", "adi_get_fields", "adi_set_source", "adi_set_point_source", "adi_step", "adi_synchronize",
    "adi_step_index", "adi_launches_per_step", "adi_stream", "adi_last_error", "adi_set_timing",
    "adi_timing_report", "adi_debug_matrices", "adi_debug_materials_tf", "adi_debug_sweep", "adi_debug_rhs_e",
    "adi_debug_rhs_h", "adi_debug_solve_e",
    "adi_box_sweep", "adi_box_factor", "adi_box_rhs", "adi_box_copy", "adi_box_abc", "adi_box_pec",
    "adi_box_materials_tf", "adi_set_sweep_order", "adi_energy", "adi_project_weighted", "adi_errors_uA", "adi_divergence",
    "adi_nccl_unique_id", "adi_loopback_create", "adi_loopback_destroy", "adi_set_zsolve", "adi_zsolve_tables",
    "adi_set_rhs_variant",
]



def build(force: bool = False, verbose: bool = False, lib_path: str | None = None, extra_flags=(),
          degrees=DEGREES) -> str:
    """Compile libadimaxwell.so in-tree for sm_100a (nvcc; no GPU needed).

    One object per B-spline degree (csrc/degree.cu with -DADI_P=p) plus the host
    orchestration (csrc/adi_maxwell.cu), compiled in parallel, then linked."""
    lib_path = lib_path or LIB_PATH
    os.makedirs(os.path.dirname(lib_path), exist_ok=True)
    newest = max(os.path.getmtime(s) for s in SOURCES)
    if not (force or not os.path.exists(lib_path) or os.path.getmtime(lib_path) < newest):
        return lib_path
    objdir = os.path.join(os.path.dirname(lib_path), "obj")
    os.makedirs(objdir, exist_ok=True)
    jobs = [(os.path.join(objdir, "adi_maxwell.o"), [os.path.join(CSRC, "adi_maxwell.cu")])]
    for p in DEGREES:  # degrees not in `degrees` (tuning builds) compile as stubs
        stub = [] if p in degrees else ["-DADI_STUB"]
        jobs.append((os.path.join(objdir, f"degree_p{p}.o"), [f"-DADI_P={p}", *stub, os.path.join(CSRC, "degree.cu")]))
    procs = []
    for obj, args in jobs:
        cmd = ["nvcc", *NVCC_FLAGS, *extra_flags, "-c", "-o", obj, *args]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
    bad = [cmd for cmd, pr in procs if pr.wait() != 0]
    if bad:
        raise RuntimeError("nvcc failed: " + " | ".join(" ".join(c) for c in bad))
    tmp = lib_path + ".tmp"
    cmd = ["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *[o for o, _ in jobs], "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib_path)
    return lib_path


class SweepJob(C.Structure):
    """adi_sweep_job (include/adi_maxwell.h)."""
    _fields_ = [("in_", C.c_void_p), ("out", C.c_void_p), ("c", C.c_void_p), ("iu", C.c_void_p),
                ("base", C.c_void_p), ("coef", C.c_double), ("dims", C.c_int64 * 3), ("axis", C.c_int32),
                ("comp", C.c_int32)]


class AdiConfig(C.Structure):
    """adi_config (include/adi_maxwell.h)."""
    _fields_ = [("n", C.c_int32), ("p", C.c_int32), ("tau", C.c_double), ("bc", C.c_int32),
                ("device", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32), ("stream", C.c_void_p),
                ("nccl_id", C.c_void_p), ("loopback", C.c_void_p)]


_lib = None
_lock = threading.Lock()
_dp = C.POINTER(C.c_double)


def lib():
    """Load libadimaxwell.so (raises if it is missing -- no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build() (nvcc, sm_100a)")
            L = C.CDLL(LIB_PATH)
            L.adi_create.argtypes = [C.POINTER(AdiConfig), C.POINTER(C.c_void_p)]
            L.adi_destroy.argtypes = [C.c_void_p]
            L.adi_destroy.restype = None
            L.adi_layout.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
            L.adi_set_tau.argtypes = [C.c_void_p, C.c_double]
            L.adi_set_materials.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_set_materials_tf.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_set_fields.argtypes = [C.c_void_p, C.c_void_p]
            L.adi_get_fields.argtypes = [C.c_void_p, C.c_void_p]
            L.adi_set_source.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
            L.adi_set_point_source.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_double,
                                               C.c_void_p, C.c_int64]
            L.adi_step.argtypes = [C.c_void_p, C.c_int64]
            L.adi_synchronize.argtypes = [C.c_void_p]
            L.adi_step_index.argtypes = [C.c_void_p]
            L.adi_step_index.restype = C.c_int64
            L.adi_launches_per_step.argtypes = [C.c_void_p]
            L.adi_launches_per_step.restype = C.c_int64
            L.adi_stream.argtypes = [C.c_void_p]
            L.adi_stream.restype = C.c_void_p
            L.adi_last_error.restype = C.c_char_p
            L.adi_set_timing.argtypes = [C.c_void_p, C.c_int32]
            L.adi_timing_report.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_debug_matrices.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_debug_materials_tf.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_debug_sweep.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
            L.adi_debug_rhs_e.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
            L.adi_debug_rhs_h.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_debug_solve_e.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
            i64x3 = C.POINTER(C.c_int64)
            L.adi_box_sweep.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(SweepJob)]
            L.adi_box_factor.argtypes = [C.c_void_p, C.c_int32, C.c_int32, i64x3, C.c_void_p, C.c_void_p]
            L.adi_box_rhs.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_double, C.c_void_p]
            L.adi_box_copy.argtypes = [C.c_void_p, C.c_void_p, i64x3, i64x3, C.c_void_p, i64x3, i64x3, i64x3]
            L.adi_box_abc.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
            L.adi_box_pec.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, i64x3, i64x3]
            L.adi_box_materials_tf.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_set_sweep_order.argtypes = [C.c_void_p, C.c_int32]
            L.adi_energy.argtypes = [C.c_void_p, C.c_void_p]
            L.adi_project_weighted.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.adi_errors_uA.argtypes = [C.c_void_p, C.c_double, C.c_void_p]
            L.adi_divergence.argtypes = [C.c_void_p, C.c_void_p]
            L.adi_nccl_unique_id.argtypes = [C.c_void_p]
            L.adi_loopback_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
            L.adi_loopback_destroy.argtypes = [C.c_void_p]
            L.adi_loopback_destroy.restype = None
            L.adi_set_zsolve.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
            L.adi_set_rhs_variant.argtypes = [C.c_void_p, C.c_int32]
            L.adi_zsolve_tables.argtypes = [C.c_int32] * 6 + [C.POINTER(C.c_int32)] * 2 + [C.c_void_p] * 4
            _lib = L
        return _lib


class AdiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"adi status {status}: {msg}")
        self.status = status


def _addr(x, count: int | None = None, what: str = "array") -> int:
    """Address of a host numpy array or a torch tensor (host or CUDA) of float64 entries.

    Raises ValueError (not assert: the checks must survive ``python -O``) unless the array is
    C-contiguous float64 and, when ``count`` is given, holds exactly ``count`` entries -- the
    library copies ``count`` doubles from / to the pointer."""
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{what}: need a C-contiguous float64 array, got {x.dtype}")
        n = x.size
        addr = x.ctypes.data
    else:  # torch.Tensor
        import torch
        if not isinstance(x, torch.Tensor):
            raise ValueError(f"{what}: need a numpy array or a torch tensor, got {type(x).__name__}")
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError(f"{what}: need a contiguous float64 tensor, got {x.dtype}")
        n = x.numel()
        addr = x.data_ptr()
    if count is not None and n != count:
        raise ValueError(f"{what}: {n} entries, expected {count}")
    return addr


def _as_f64(x):
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    return x


def _ptr_array(objs, count: int | None = None, what: str = "array"):
    arr = (C.c_void_p * len(objs))()
    for i, o in enumerate(objs):
        arr[i] = None if o is None else _addr(o, count, f"{what}[{i}]")
    return arr


def nccl_unique_id() -> bytes:
    """Rank 0 of a distributed run: a fresh 128-byte ncclUniqueId (adi_nccl_unique_id), to be
    broadcast to every rank and passed to Patch(..., nccl_id=...)."""
    L = lib()
    buf = C.create_string_buffer(128)
    st = L.adi_nccl_unique_id(buf)
    if st != ADI_OK:
        raise AdiError(st, L.adi_last_error().decode())
    return buf.raw


class Loopback:
    """In-process exchange group of `nranks` patches driven by `nranks` host threads on one
    device (adi_loopback_create): the library's distributed schedule without NCCL."""

    def __init__(self, nranks: int):
        self._L = lib()
        h = C.c_void_p()
        st = self._L.adi_loopback_create(int(nranks), C.byref(h))
        if st != ADI_OK:
            raise AdiError(st, self._L.adi_last_error().decode())
        self.h = h
        self.nranks = int(nranks)

    def close(self):
        if getattr(self, "h", None):
            self._L.adi_loopback_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Patch:
    """One n x n x n patch (or, distributed, this rank's z-slab of it) on one B200; device
    memory owned by the library.  nranks > 1 with nccl_id (bytes from nccl_unique_id()) or
    loopback (a Loopback group) runs the library's distributed schedule; nranks > 1 with
    neither is a box-mode patch (adi_box_* only)."""

    def __init__(self, n: int, p: int, tau: float, bc: int = ADI_BC_PEC, device: int = 0, rank: int = 0,
                 nranks: int = 1, stream: int | None = None, nccl_id: bytes | None = None,
                 loopback: "Loopback | None" = None):
        L = lib()
        self._L = L
        self._id = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id: need the 128-byte ncclUniqueId")
            self._id = C.create_string_buffer(bytes(nccl_id), 128)
        self._loop = loopback
        cfg = AdiConfig(int(n), int(p), float(tau), int(bc), int(device), int(rank), int(nranks), stream,
                        C.cast(self._id, C.c_void_p) if self._id is not None else None,
                        loopback.h if loopback is not None else None)
        h = C.c_void_p()
        self._check(L.adi_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.n, self.p, self.tau, self.bc = int(n), int(p), float(tau), int(bc)
        self.N = self.n + self.p
        self.U = self.N ** 3

    def _check(self, st: int):
        if st != ADI_OK:
            raise AdiError(st, self._L.adi_last_error().decode())

    def close(self):
        if getattr(self, "h", None):
            self._L.adi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- setup -------------------------------------------------------------
    def set_tau(self, tau: float):
        self._check(self._L.adi_set_tau(self.h, float(tau)))
        self.tau = float(tau)

    @property
    def local_count(self) -> int:
        """Entries of one field held by this patch (the local slab N x N x (k1 - k0))."""
        N, k0, k1 = self.layout()
        return N * N * (k1 - k0)

    def set_materials(self, eps_elem, mu_elem=None):
        ne = self.n ** 3
        e, m = _as_f64(eps_elem), (None if mu_elem is None else _as_f64(mu_elem))
        self._check(self._L.adi_set_materials(self.h, _addr(e, ne, "eps_elem"),
                                              None if m is None else _addr(m, ne, "mu_elem")))

    def set_materials_tf(self, eps_tf, mu_tf=None):
        e, m = _as_f64(eps_tf), (None if mu_tf is None else _as_f64(mu_tf))
        self._check(self._L.adi_set_materials_tf(self.h, _addr(e, self.U, "eps_tf"),
                                                 None if m is None else _addr(m, self.U, "mu_tf")))

    def set_fields(self, fields):
        fs = [_as_f64(f) for f in fields]
        if len(fs) != 6:
            raise ValueError(f"set_fields: need 6 fields, got {len(fs)}")
        self._check(self._L.adi_set_fields(self.h, _ptr_array(fs, self.local_count, "fields")))

    def get_fields(self, out=None):
        if out is None:
            out = [np.empty(self.local_count) for _ in range(6)]
        if len(out) != 6:
            raise ValueError(f"get_fields: need 6 output arrays, got {len(out)}")
        self._check(self._L.adi_get_fields(self.h, _ptr_array(out, self.local_count, "out")))
        return out

    def set_source(self, loads, signal):
        if len(loads) != 3:
            raise ValueError("set_source: need 3 load vectors (or None)")
        ls = [None if l is None else _as_f64(l) for l in loads]
        sig = _as_f64(signal)
        self._check(self._L.adi_set_source(self.h, _ptr_array(ls, self.U, "loads"), _addr(sig, None, "signal"),
                                           int(len(sig))))

    def set_point_source(self, comp: int, pos, signal):
        sig = _as_f64(signal)
        self._check(self._L.adi_set_point_source(self.h, int(comp), float(pos[0]), float(pos[1]), float(pos[2]),
                                                 _addr(sig), int(len(sig))))

    # ---- stepping ------------------------------------------------------------
    def step(self, k: int = 1):
        self._check(self._L.adi_step(self.h, int(k)))

    def synchronize(self):
        self._check(self._L.adi_synchronize(self.h))

    @property
    def step_index(self) -> int:
        return int(self._L.adi_step_index(self.h))

    @property
    def launches_per_step(self) -> int:
        return int(self._L.adi_launches_per_step(self.h))

    @property
    def stream(self) -> int:
        return int(self._L.adi_stream(self.h) or 0)

    def set_sweep_order(self, order: int):
        """0: stiffened axis first (D7, default); 1: paper-literal x -> y -> z (V1)."""
        self._check(self._L.adi_set_sweep_order(self.h, int(order)))

    def set_rhs_variant(self, variant: int):
        """NEXT-2: 0 = row factors of the test function on the E right-hand sides (D5, default);
        2 = element-wise material inside their quadrature (V2)."""
        self._check(self._L.adi_set_rhs_variant(self.h, int(variant)))

    def set_zsolve(self, mode: int) -> bool:
        """NEXT-1: 1 (default) partitioned (SPIKE) z-solve of the constant sweeps of a distributed
        patch; 0: every z sweep between transposes.  Returns whether the partitioned solve is in effect."""
        act = C.c_int32(0)
        self._check(self._L.adi_set_zsolve(self.h, int(mode), C.byref(act)))
        return bool(act.value)

    def energy(self):
        """(per-field f^T M^3 f [6], M-norm energy 1/2 sum) -- on-device diagnostic."""
        out = (C.c_double * 7)()
        self._check(self._L.adi_energy(self.h, out))
        return [out[c] for c in range(6)], out[6]

    def errors_uA(self, t: float):
        """(||E_h-E||_L2, ||H_h-H||_L2, ||E_h-E||_Hcurl, ||H_h-H||_Hcurl) against u_A(., t)."""
        out = (C.c_double * 4)()
        self._check(self._L.adi_errors_uA(self.h, float(t), out))
        return [out[k] for k in range(4)]

    def divergence(self):
        """(||div E_h||_L2, ||div H_h||_L2) of the current fields."""
        out = (C.c_double * 2)()
        self._check(self._L.adi_divergence(self.h, out))
        return [out[0], out[1]]

    def project_weighted(self, f, eps_tf, out=None):
        """NEXT-4 (Appendix): u with diag(eps^)(M (x) M (x) M) u = f.  f, eps_tf: CUDA
        float64 tensors of N^3 entries (x fastest); out (default: a new tensor) may be f.
        Asynchronous on the patch stream."""
        import torch
        if out is None:
            out = torch.empty_like(f)
        for t in (f, eps_tf, out):
            assert t.is_cuda and t.numel() == self.N ** 3, "need CUDA tensors of N^3 entries"
        self._check(self._L.adi_project_weighted(self.h, _addr(f), _addr(eps_tf), _addr(out)))
        return out

    def set_timing(self, enable: bool):
        self._check(self._L.adi_set_timing(self.h, int(bool(enable))))

    def timing_report(self):
        ms = (C.c_double * len(K_CLASSES))()
        n = (C.c_int64 * len(K_CLASSES))()
        self._check(self._L.adi_timing_report(self.h, ms, n))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(K_CLASSES)}

    def layout(self):
        """(N, k0, k1): this rank's z-slab [k0, k1) of the N^3 grid."""
        N, k0, k1 = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self._L.adi_layout(self.h, C.byref(N), C.byref(k0), C.byref(k1)))
        return N.value, k0.value, k1.value

    # ---- box-level calls (slab-decomposed path; torch CUDA tensors) ---------------
    @staticmethod
    def _i3(v):
        return (C.c_int64 * 3)(*[int(x) for x in v])

    def box_sweep(self, mode: int, jobs):
        """jobs: list of dicts with keys in, out, dims, axis, comp [, c, iu, base, coef]."""
        arr = (SweepJob * len(jobs))()
        for a, j in zip(arr, jobs):
            a.in_ = _addr(j["in"])
            a.out = _addr(j["out"])
            a.c = _addr(j["c"]) if j.get("c") is not None else None
            a.iu = _addr(j["iu"]) if j.get("iu") is not None else None
            a.base = _addr(j["base"]) if j.get("base") is not None else None
            a.coef = float(j.get("coef", 0.0))
            a.dims = (C.c_int64 * 3)(*[int(x) for x in j["dims"]])
            a.axis = int(j["axis"])
            a.comp = int(j["comp"])
        self._check(self._L.adi_box_sweep(self.h, int(mode), len(jobs), arr))

    def box_factor(self, comp: int, axis: int, dims, c, iu):
        self._check(self._L.adi_box_factor(self.h, int(comp), int(axis), self._i3(dims), _addr(c), _addr(iu)))

    def box_rhs(self, kind: int, s: int, d: int, ins, nzin: int, zoff: int, kg0: int, nzout: int, a, b, c, load,
                sval: float, out):
        self._check(self._L.adi_box_rhs(self.h, int(kind), int(s), int(d), _ptr_array(list(ins) + [None] * (4 - len(ins))),
                                        int(nzin), int(zoff), int(kg0), int(nzout),
                                        None if a is None else _addr(a), None if b is None else _addr(b),
                                        None if c is None else _addr(c), None if load is None else _addr(load),
                                        float(sval), _addr(out)))

    def box_copy(self, dst, ddims, doff, src, sdims, soff, ext):
        self._check(self._L.adi_box_copy(self.h, _addr(dst), self._i3(ddims), self._i3(doff), _addr(src),
                                         self._i3(sdims), self._i3(soff), self._i3(ext)))

    def box_abc(self, eps_tf, mu_tf, count: int, a, b, c):
        self._check(self._L.adi_box_abc(self.h, _addr(eps_tf), _addr(mu_tf), int(count), _addr(a), _addr(b), _addr(c)))

    def box_pec(self, comp: int, u, dims, off):
        self._check(self._L.adi_box_pec(self.h, int(comp), _addr(u), self._i3(dims), self._i3(off)))

    def box_materials_tf(self, eps_elem, mu_elem, eps_tf, mu_tf):
        e = _as_f64(eps_elem)
        m = None if mu_elem is None else _as_f64(mu_elem)
        self._check(self._L.adi_box_materials_tf(self.h, _addr(e), None if m is None else _addr(m), _addr(eps_tf),
                                                 _addr(mu_tf)))

    # ---- test-only -------------------------------------------------------------
    def matrices(self):
        N = self.N
        M, S, A = (np.zeros((N, N)) for _ in range(3))
        self._check(self._L.adi_debug_matrices(self.h, _addr(M), _addr(S), _addr(A)))
        return M, S, A

    def materials_tf(self):
        e, m = np.zeros(self.U), np.zeros(self.U)
        self._check(self._L.adi_debug_materials_tf(self.h, _addr(e), _addr(m)))
        return e, m

    def sweep(self, comp: int, axis: int, modified: bool, rhs):
        r = _as_f64(rhs)
        out = np.zeros(self.U)
        self._check(self._L.adi_debug_sweep(self.h, int(comp), int(axis), int(bool(modified)), _addr(r, self.U, "rhs"),
                                            _addr(out)))
        return out

    def solve_e(self, s: int, d: int, rhs):
        r = _as_f64(rhs)
        out = np.zeros(self.U)
        self._check(self._L.adi_debug_solve_e(self.h, int(s), int(d), _addr(r, self.U, "rhs"), _addr(out)))
        return out

    def rhs_e(self, s: int):
        R = [np.zeros(self.U) for _ in range(3)]
        self._check(self._L.adi_debug_rhs_e(self.h, int(s), _ptr_array(R)))
        return R

    def rhs_h(self, s: int, Eo, En):
        G = [np.zeros(self.U) for _ in range(3)]
        eo = [_as_f64(x) for x in Eo]
        en = [_as_f64(x) for x in En]
        self._check(self._L.adi_debug_rhs_h(self.h, int(s), _ptr_array(eo), _ptr_array(en), _ptr_array(G)))
        return G


def zsolve_tables(n: int, p: int, nranks: int, rank: int, lo: int, hi: int):
    """Host tables of the NEXT-1 partitioned z-solve (adi_zsolve_tables; no device needed):
    dict(g0, m, fac [m, 2p+1], tw [2p, m], C [p, p], B [p, p], q [2p, 2p nranks])."""
    L = lib()
    N = n + p
    W = 2 * p + 1
    fac = np.zeros(N * W)
    tw = np.zeros(2 * p * N)
    cb = np.zeros(2 * p * p)
    q = np.zeros(2 * p * 2 * p * nranks)
    g0, m = C.c_int32(0), C.c_int32(0)
    st = L.adi_zsolve_tables(n, p, nranks, rank, lo, hi, C.byref(g0), C.byref(m), fac.ctypes.data, tw.ctypes.data,
                             cb.ctypes.data, q.ctypes.data)
    if st != ADI_OK:
        raise AdiError(st, L.adi_last_error().decode())
    mm = m.value
    return dict(g0=g0.value, m=mm, fac=fac[:mm * W].reshape(mm, W).copy(), tw=tw[:2 * p * mm].reshape(2 * p, mm).copy(),
                C=cb[:p * p].reshape(p, p).copy(), B=cb[p * p:].reshape(p, p).copy(),
                q=q.reshape(2 * p, 2 * p * nranks).copy())
