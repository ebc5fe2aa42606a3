"""CPU oracle for the ADI isogeometric Maxwell step (arXiv 2103.06998).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2103_06998_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``adi_oracle.c`` (plain C, fp64, single thread unless
``Patch.set_threads`` asks for more, ``-O2 -ffp-contract=off``); this module is ctypes marshalling only.
Every function of the C file cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "adi_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_dp = C.POINTER(C.c_double)


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (gcc, plain C)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            L.orc_create.restype = C.c_void_p
            L.orc_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int]
            L.orc_destroy.argtypes = [C.c_void_p]
            L.orc_last_error.restype = C.c_char_p
            L.orc_max_growth.restype = C.c_double
            L.orc_max_growth.argtypes = [C.c_void_p]
            L.orc_step_index.restype = C.c_int64
            L.orc_step_index.argtypes = [C.c_void_p]
            L.orc_step.argtypes = [C.c_void_p, C.c_int64]
            L.orc_set_tau.argtypes = [C.c_void_p, C.c_double]
            L.orc_basis.argtypes = [C.c_void_p, C.c_double, _dp, _dp]
            L.orc_exact_uA.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, _dp, _dp]
            L.orc_errors_uA.argtypes = [C.c_void_p, C.c_double, _dp]
            L.orc_project_uA.argtypes = [C.c_void_p, C.c_double]
            L.orc_project_weighted.argtypes = [C.c_void_p, _dp, _dp, _dp]
            L.orc_point_load.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, _dp]
            L.orc_set_source.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_int64]
            L.orc_set_rhs_variant.argtypes = [C.c_void_p, C.c_int]
            L.orc_set_threads.argtypes = [C.c_void_p, C.c_int]
            _lib = L
        return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _arr6(arrs):
    P6 = _dp * len(arrs)
    return P6(*[_ptr(a) if a is not None else _dp() for a in arrs])


class OracleError(RuntimeError):
    pass


class Patch:
    """One n x n x n patch of degree-p C^{p-1} B-splines (host, fp64)."""

    def __init__(self, n: int, p: int, tau: float, bc: int = 0):
        L = lib()
        self._L = L
        h = L.orc_create(int(n), int(p), float(tau), int(bc))
        if not h:
            raise OracleError(L.orc_last_error().decode())
        self.h = C.c_void_p(h)
        self.n, self.p, self.tau, self.bc = int(n), int(p), float(tau), int(bc)
        self.N = self.n + self.p
        self.U = self.N ** 3

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._L.orc_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            raise OracleError(f"status {st}: {self._L.orc_last_error().decode()}")

    # -- setup ---------------------------------------------------------------
    def knots(self):
        t = np.zeros(self.n + 2 * self.p + 1)
        self._L.orc_knots(self.h, _ptr(t))
        return t

    def matrices(self):
        N = self.N
        M, S, A = (np.zeros((N, N)) for _ in range(3))
        self._L.orc_matrices(self.h, _ptr(M), _ptr(S), _ptr(A))
        return M, S, A

    def basis(self, x: float):
        v, d = np.zeros(self.N), np.zeros(self.N)
        self._L.orc_basis(self.h, float(x), _ptr(v), _ptr(d))
        return v, d

    def material_weights(self):
        w = np.zeros((self.N, self.n))
        self._L.orc_material_weights(self.h, _ptr(w))
        return w

    def set_tau(self, tau: float):
        self._check(self._L.orc_set_tau(self.h, C.c_double(tau)))
        self.tau = float(tau)

    def set_materials(self, eps_e, mu_e=None):
        e = np.ascontiguousarray(eps_e, dtype=np.float64).reshape(-1)
        m = None if mu_e is None else np.ascontiguousarray(mu_e, dtype=np.float64).reshape(-1)
        assert e.size == self.n ** 3
        self._check(self._L.orc_set_materials(self.h, _ptr(e), _ptr(m) if m is not None else _dp()))

    def set_materials_tf(self, eps_tf, mu_tf=None):
        e = np.ascontiguousarray(eps_tf, dtype=np.float64).reshape(-1)
        m = None if mu_tf is None else np.ascontiguousarray(mu_tf, dtype=np.float64).reshape(-1)
        assert e.size == self.U
        self._check(self._L.orc_set_materials_tf(self.h, _ptr(e), _ptr(m) if m is not None else _dp()))

    def get_materials_tf(self):
        e, m = np.zeros(self.U), np.zeros(self.U)
        self._L.orc_get_materials_tf(self.h, _ptr(e), _ptr(m))
        return e, m

    def set_fields(self, fields):
        fs = [np.ascontiguousarray(f, dtype=np.float64).reshape(-1) for f in fields]
        assert len(fs) == 6 and all(f.size == self.U for f in fs)
        self._check(self._L.orc_set_fields(self.h, _arr6(fs)))

    def get_fields(self):
        fs = [np.zeros(self.U) for _ in range(6)]
        self._check(self._L.orc_get_fields(self.h, _arr6(fs)))
        return fs

    def set_source(self, loads, signal):
        ls = [None if l is None else np.ascontiguousarray(l, dtype=np.float64).reshape(-1) for l in loads]
        sig = np.ascontiguousarray(signal, dtype=np.float64).reshape(-1)
        self._keep = (ls, sig)
        arr = _arr6(ls)
        self._check(self._L.orc_set_source(self.h, C.cast(arr, C.c_void_p), _ptr(sig), C.c_int64(sig.size)))

    def point_load(self, x, y, z):
        out = np.zeros(self.U)
        self._L.orc_point_load(self.h, float(x), float(y), float(z), _ptr(out))
        return out

    # -- stepping --------------------------------------------------------------
    def step(self, k: int = 1):
        self._check(self._L.orc_step(self.h, C.c_int64(k)))

    @property
    def step_index(self) -> int:
        return int(self._L.orc_step_index(self.h))

    def set_order_variant(self, v: int):
        self._L.orc_set_order_variant(self.h, int(v))

    def set_threads(self, t: int):
        """Split the independent-output loops (kron3 output points, sweep fibers) over t OpenMP
        threads; results are bit-identical to the default single thread."""
        self._L.orc_set_threads(self.h, int(t))

    def set_rhs_variant(self, v: int):
        """0: material of the test function on the RHS rows (D5); 2: element-wise material inside
        the RHS quadrature (V2, NEXT-2; needs set_materials with element values)."""
        self._L.orc_set_rhs_variant(self.h, int(v))

    @property
    def max_growth(self) -> float:
        return float(self._L.orc_max_growth(self.h))

    # -- debug / per-stage entry points ---------------------------------------
    def rhs_e(self, s: int):
        R = [np.zeros(self.U) for _ in range(3)]
        self._check(self._L.orc_debug_rhs_e(self.h, int(s), _arr6(R)))
        return R

    def rhs_h(self, s: int, Eo, En):
        G = [np.zeros(self.U) for _ in range(3)]
        Eo = [np.ascontiguousarray(x, dtype=np.float64) for x in Eo]
        En = [np.ascontiguousarray(x, dtype=np.float64) for x in En]
        self._check(self._L.orc_debug_rhs_h(self.h, int(s), _arr6(Eo), _arr6(En), _arr6(G)))
        return G

    def solve_e(self, s: int, d: int, rhs):
        u = np.array(rhs, dtype=np.float64, copy=True).reshape(-1)
        self._check(self._L.orc_debug_solve_e(self.h, int(s), int(d), _ptr(u)))
        return u

    def sweep(self, comp: int, axis: int, modified: bool, rhs):
        u = np.array(rhs, dtype=np.float64, copy=True).reshape(-1)
        self._check(self._L.orc_debug_sweep(self.h, int(comp), int(axis), int(bool(modified)), _ptr(u)))
        return u

    def sweep_c(self, comp: int, axis: int, c, rhs):
        u = np.array(rhs, dtype=np.float64, copy=True).reshape(-1)
        cc = np.ascontiguousarray(c, dtype=np.float64).reshape(-1)
        self._check(self._L.orc_debug_sweep_c(self.h, int(comp), int(axis), _ptr(cc), _ptr(u)))
        return u

    def kron(self, ox: int, oy: int, oz: int, u):
        """(X (x) Y (x) Z) u with codes 0=M, 1=A, 2=B=A^T, 3=S."""
        uu = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        out = np.zeros(self.U)
        self._L.orc_debug_kron(self.h, int(ox), int(oy), int(oz), _ptr(uu), _ptr(out))
        return out

    # -- manufactured solution --------------------------------------------------
    def project_uA(self, t: float = 0.0):
        self._check(self._L.orc_project_uA(self.h, float(t)))

    def project_weighted(self, f, eps_tf):
        """NEXT-4 (Appendix): u with diag(eps)(M (x) M (x) M) u = f."""
        ff = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        ee = np.ascontiguousarray(eps_tf, dtype=np.float64).reshape(-1)
        u = np.zeros(self.U)
        self._check(self._L.orc_project_weighted(self.h, _ptr(ff), _ptr(ee), _ptr(u)))
        return u

    def errors_uA(self, t: float):
        out = np.zeros(4)
        self._L.orc_errors_uA(self.h, float(t), _ptr(out))
        return out


def exact_uA(x, y, z, t):
    """u_A (P:286-318 with D8): returns (fields[6], curls[6])."""
    L = lib()
    out, cu = np.zeros(6), np.zeros(6)
    L.orc_exact_uA(float(x), float(y), float(z), float(t), _ptr(out), _ptr(cu))
    return out, cu
