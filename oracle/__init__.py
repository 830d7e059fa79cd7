"""TEST INFRASTRUCTURE ONLY — CPU checkers for the B200 hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg
and ``--impl reference`` arm) may import this package, and only as the checker
or the timed CPU baseline — never as the product path.

Two interchangeable backends with one Python surface:

* ``port()``  — ``oracle/liboracle_port.so``, the plain-C restatement in
  ``oracle/skr_oracle.c`` (every function cites the reference file:line).
* ``ref()``   — ``oracle/_ref/libskridge_ref.so``, the UNMODIFIED reference
  library compiled from /root/reference/proj/src plus the extern "C" shim
  ``oracle/ref_capi.cpp``.  Present wherever it was built (it travels to the GPU
  box with the repo snapshot); ``ref_available()`` says whether it loaded.

Array conventions: X is (n, d) C-contiguous float64 (== the reference's d x n
column-major DenseMatrix); U is returned as (d, k) with Fortran order, i.e.
column j is basis vector j exactly as DenseMatrix stores it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "liboracle_port.so")
REF_PATH = os.path.join(_HERE, "_ref", "libskridge_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64, u64, f64, cint = C.c_int64, C.c_uint64, C.c_double, C.c_int
vp = C.c_void_p
P = C.POINTER

ERRORS = {1: "DimensionError", 2: "ParameterError", 3: "InputError", 4: "ScaleGuardError",
          5: "DivergenceError", 8: "EmptyBasisError", 10: "InternalError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


@dataclass
class Sketch:
    U: np.ndarray          # (d, k) column-major basis
    sigma: np.ndarray      # (k,)
    V: np.ndarray | None   # (n, k) or None
    k: int
    q: int
    rank_reduced: bool


@dataclass
class SvrgOut:
    iterate: np.ndarray
    trace: np.ndarray
    diverged: bool = False
    error: str = ""


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _Backend:
    """Common wrapper; `prefix` is "skro_" (port) or "ref_" (reference shim)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.name = "port" if prefix == "skro_" else "reference"
        self._err = self._fn("last_error", C.c_char_p, [])

    def _fn(self, name, res, args):
        f = getattr(self.lib, self.prefix + name)
        f.restype = res
        f.argtypes = args
        return f

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    # -- random.cpp --------------------------------------------------------
    def uniforms(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count)
        self._check(self._fn("uniforms", cint, [u64, i64, _dp])(seed, count, out))
        return out

    def gaussian_matrix(self, rows: int, cols: int, seed: int) -> np.ndarray:
        """(rows, cols) array whose Fortran-order bytes equal the reference DenseMatrix."""
        out = np.empty(rows * cols)
        self._check(self._fn("gaussian_matrix", cint, [i64, i64, u64, _dp])(rows, cols, seed, out))
        return out.reshape(cols, rows).T

    def sym_eigs(self, a: np.ndarray):
        n = a.shape[0]
        vals = np.empty(n)
        vecs = np.empty(n * n)
        self._check(self._fn("sym_eigs", cint, [_dp, i64, _dp, _dp])(
            _c64(np.asfortranarray(a).ravel(order="F")), n, vals, vecs))
        return vals, vecs.reshape(n, n).T

    # -- sketch.cpp --------------------------------------------------------
    def block_lanczos(self, x, k, q=0, seed=0, scale=None, eps_prime=0.5, want_right=True):
        x = _c64(x)
        n, d = x.shape
        if scale is None:
            scale = 1.0 / math.sqrt(n)
        U = np.zeros(d * k)
        sig = np.zeros(k)
        V = np.zeros(n * k) if want_right else None
        ku, qu = i64(), i64()
        rr = cint()
        if self.prefix == "skro_":
            f = self._fn("block_lanczos", cint, [_dp, i64, i64, f64, i64, i64, f64, u64, _dp, _dp,
                                                  vp, P(i64), P(i64), P(cint), P(i64)])
            rc = f(x, n, d, scale, k, q, eps_prime, seed, U, sig,
                   V.ctypes.data if V is not None else None, C.byref(ku), C.byref(qu),
                   C.byref(rr), None)
        else:
            f = self._fn("block_lanczos", cint, [_dp, i64, i64, f64, i64, i64, f64, u64, _dp, _dp,
                                                  vp, P(i64), P(i64), P(cint)])
            rc = f(x, n, d, scale, k, q, eps_prime, seed, U, sig,
                   V.ctypes.data if V is not None else None, C.byref(ku), C.byref(qu), C.byref(rr))
        self._check(rc)
        kk = ku.value
        Um = U[: d * kk].reshape(kk, d).T
        Vm = V[: n * kk].reshape(kk, n).T if V is not None else None
        return Sketch(Um, sig[:kk].copy(), Vm, kk, qu.value, bool(rr.value))

    # -- sparse inputs (reference backend only): (row_ptr, col_idx, vals, d) CSR over
    #    points == the reference's CSC over points (sparse_matrix.hpp:8-14) ---------
    @staticmethod
    def _csr(csr):
        rp, ci, va, d = csr
        return (np.ascontiguousarray(rp, dtype=np.int64), np.ascontiguousarray(ci, dtype=np.int32), _c64(va),
                len(rp) - 1, int(d))

    def block_lanczos_csr(self, csr, k, q=0, seed=0, scale=None, eps_prime=0.5, want_right=True):
        if self.prefix == "skro_":
            raise NotImplementedError("sparse inputs: reference backend only")
        rp, ci, va, n, d = self._csr(csr)
        scale = 1.0 / math.sqrt(n) if scale is None else scale
        U, sig = np.zeros(d * k), np.zeros(k)
        V = np.zeros(n * k) if want_right else None
        ku, qu, rr = i64(), i64(), cint()
        ip64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
        ip32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
        f = self._fn("block_lanczos_csr", cint, [ip64, ip32, _dp, i64, i64, f64, i64, i64, f64, u64, _dp, _dp,
                                                 vp, P(i64), P(i64), P(cint)])
        self._check(f(rp, ci, va, n, d, scale, k, q, eps_prime, seed, U, sig,
                      V.ctypes.data if V is not None else None, C.byref(ku), C.byref(qu), C.byref(rr)))
        kk = ku.value
        return Sketch(U[: d * kk].reshape(kk, d).T, sig[:kk].copy(),
                      V[: n * kk].reshape(kk, n).T if V is not None else None, kk, qu.value, bool(rr.value))

    def objective_csr(self, csr, y, lam, w) -> float:
        rp, ci, va, n, d = self._csr(csr)
        ip64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
        ip32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
        out = f64()
        self._check(self._fn("objective_csr", cint, [ip64, ip32, _dp, i64, i64, _dp, f64, _dp, P(f64)])(
            rp, ci, va, n, d, _c64(y), lam, _c64(w), C.byref(out)))
        return out.value

    def reference_minimum_csr(self, csr, y, lam):
        rp, ci, va, n, d = self._csr(csr)
        ip64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
        ip32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
        w, mn = np.empty(d), f64()
        self._check(self._fn("reference_minimum_csr", cint, [ip64, ip32, _dp, i64, i64, _dp, f64, _dp, P(f64)])(
            rp, ci, va, n, d, _c64(y), lam, w, C.byref(mn)))
        return w, mn.value

    def problem_csr(self, csr, y, lam, U=None, sigma=None, mode=2) -> "Problem":
        """PreconditionedRidge over sparse data; mode 0 Dense, 1 Lazy, 2 Auto (ridge.hpp:121-123)."""
        if self.prefix == "skro_":
            raise NotImplementedError("sparse inputs: reference backend only")
        return Problem(self, None, y, lam, U, sigma, mode, csr=csr)

    # -- ridge.cpp / bench.cpp / precond.cpp -----------------------------------
    def objective(self, x, y, lam, w) -> float:
        x = _c64(x)
        n, d = x.shape
        out = f64()
        self._check(self._fn("objective", cint, [_dp, i64, i64, _dp, f64, _dp, P(f64)])(
            x, n, d, _c64(y), lam, _c64(w), C.byref(out)))
        return out.value

    def reference_minimum(self, x, y, lam):
        x = _c64(x)
        n, d = x.shape
        w = np.empty(d)
        mn = f64()
        self._check(self._fn("reference_minimum", cint, [_dp, i64, i64, _dp, f64, _dp, P(f64)])(
            x, n, d, _c64(y), lam, w, C.byref(mn)))
        return w, mn.value

    def reference_minimum_cg(self, x, y, lam, tol, max_it):
        """bench.cpp:56-82 (reference backend only)."""
        x = _c64(x)
        n, d = x.shape
        w = np.empty(d)
        self._check(self._fn("reference_minimum_cg", cint, [_dp, i64, i64, _dp, f64, f64, i64, _dp])(
            x, n, d, _c64(y), lam, tol, max_it, w))
        return w

    def conditioned_cond(self, x, lam, U, sigma, unguarded=False) -> float:
        x = _c64(x)
        n, d = x.shape
        k = 0 if U is None else U.shape[1]
        Uf = _c64(np.asarray(U).ravel(order="F")) if k else np.zeros(1)
        out = f64()
        if self.prefix == "skro_":
            D, c = self.build_sketched(sigma, lam) if k else (np.zeros(1), 1.0)
            self._check(self._fn("conditioned_cond", cint, [_dp, i64, i64, f64, _dp, _dp, i64, f64,
                                                             cint, P(f64)])(
                x, n, d, lam, Uf, _c64(D), k, c, int(unguarded), C.byref(out)))
        else:
            s = _c64(sigma) if k else np.zeros(1)
            self._check(self._fn("conditioned_cond", cint, [_dp, i64, i64, f64, _dp, _dp, i64, cint,
                                                             P(f64)])(
                x, n, d, lam, Uf, s, k, int(unguarded), C.byref(out)))
        return out.value

    def generate_synthetic(self, n, d, decay, noise_std, seed, normalize_columns=True):
        """dataset.cpp:16-79 (reference backend only): (X n x d, y)."""
        if self.prefix == "skro_":
            raise NotImplementedError("generate_synthetic: reference backend only")
        X = np.empty((n, d))
        y = np.empty(n)
        self._check(self._fn("generate_synthetic", cint, [i64, i64, cint, f64, u64, cint, _dp, _dp])(
            n, d, decay, noise_std, seed, int(normalize_columns), X, y))
        return X, y

    def read_sparse_corpus(self, path):
        """dataset.cpp:87-162 (reference backend only): (row_ptr, col_idx, vals, d), labels."""
        if self.prefix == "skro_":
            raise NotImplementedError("read_sparse_corpus: reference backend only")
        n, d, nnz = i64(), i64(), i64()
        p = path.encode()
        self._check(self._fn("read_corpus_sizes", cint, [C.c_char_p, P(i64), P(i64), P(i64)])(
            p, C.byref(n), C.byref(d), C.byref(nnz)))
        rp = np.empty(n.value + 1, dtype=np.int64)
        ci = np.empty(max(nnz.value, 1), dtype=np.int32)
        va = np.empty(max(nnz.value, 1))
        y = np.empty(n.value)
        ip64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
        ip32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
        self._check(self._fn("read_corpus", cint, [C.c_char_p, ip64, ip32, _dp, _dp])(p, rp, ci, va, y))
        return (rp, ci[: nnz.value], va[: nnz.value], d.value), y

    # ratio diagnostics: the unmodified reference only (no C restatement)
    def dataset_spectrum(self, x, lam) -> np.ndarray:
        if self.prefix == "skro_":
            raise NotImplementedError("dataset_spectrum: reference backend only")
        x = _c64(x)
        n, d = x.shape
        out = np.empty(d)
        self._check(self._fn("dataset_spectrum", cint, [_dp, i64, i64, f64, _dp])(x, n, d, lam, out))
        return out

    def theoretical_ratio(self, eigs, lam, k) -> float:
        if self.prefix == "skro_":
            raise NotImplementedError("theoretical_ratio: reference backend only")
        e = _c64(eigs)
        out = f64()
        self._check(self._fn("theoretical_ratio", cint, [_dp, i64, f64, i64, P(f64)])(e, len(e), lam, k,
                                                                                    C.byref(out)))
        return out.value

    def avg_condition_number(self, eigs, lam) -> float:
        if self.prefix == "skro_":
            raise NotImplementedError("avg_condition_number: reference backend only")
        e = _c64(eigs)
        out = f64()
        self._check(self._fn("avg_condition_number", cint, [_dp, i64, f64, P(f64)])(e, len(e), lam,
                                                                                  C.byref(out)))
        return out.value

    def build_sketched(self, sigma, lam):
        sigma = _c64(sigma)
        return build_sketched(sigma, lam)

    def apply_inv_sqrt(self, U, sigma, lam, v):
        d = len(v)
        k = 0 if U is None else U.shape[1]
        Uf = _c64(np.asarray(U).ravel(order="F")) if k else np.zeros(1)
        out = np.empty(d)
        if self.prefix == "skro_":
            D, c = build_sketched(sigma, lam) if k else (np.zeros(1), 1.0)
            self._check(self._fn("apply_inv_sqrt", cint, [i64, _dp, _dp, i64, f64, _dp, _dp])(
                d, Uf, _c64(D), k, c, _c64(v), out))
        else:
            s = _c64(sigma) if k else np.zeros(1)
            self._check(self._fn("apply_inv_sqrt", cint, [i64, _dp, _dp, i64, f64, _dp, _dp])(
                d, Uf, s, k, lam, _c64(v), out))
        return out

    def problem(self, x, y, lam, U=None, sigma=None, mode=0) -> "Problem":
        return Problem(self, x, y, lam, U, sigma, mode)

    def index_stream(self, betas, seed, count) -> np.ndarray:
        b = _c64(betas)
        out = np.empty(count, dtype=np.int64)
        self._check(self._fn("index_stream", cint, [_dp, i64, u64, i64, _ip])(
            b, len(b), seed, count, out))
        return out

    def cumulative_weights(self, betas) -> np.ndarray:
        b = _c64(betas)
        out = np.empty(len(b))
        self._check(self._fn("cumulative_weights", cint, [_dp, i64, _dp])(b, len(b), out))
        return out


def build_sketched(sigma, lam):
    """precond.cpp:120-136 restated on the host (k scalars)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    D = 1.0 / np.sqrt(sigma * sigma + lam)
    return D, float(D[-1])


class Problem:
    """PreconditionedRidge (Dense mode for the port; any mode for the reference)."""

    def __init__(self, be: _Backend, x, y, lam, U, sigma, mode, csr=None):
        self.be = be
        if csr is not None:
            rp, ci, va, self.n, self.d = _Backend._csr(csr)
        else:
            x = _c64(x)
            self.n, self.d = x.shape
        self.k = 0 if U is None else U.shape[1]
        self.lam = lam
        Uf = _c64(np.asarray(U).ravel(order="F")) if self.k else np.zeros(1)
        h = vp()
        if csr is not None:
            s = _c64(sigma) if self.k else np.zeros(1)
            ip64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
            ip32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
            be._check(be._fn("problem_create_csr", cint, [ip64, ip32, _dp, i64, i64, _dp, f64, _dp, _dp, i64, cint,
                                                          P(vp)])(
                rp, ci, va, self.n, self.d, _c64(y), lam, Uf, s, self.k, mode, C.byref(h)))
            self._destroy = be._fn("problem_destroy", cint, [vp])
        elif be.prefix == "skro_":
            D, c = build_sketched(sigma, lam) if self.k else (np.zeros(1), 1.0)
            be._check(be._fn("problem_create", cint, [_dp, i64, i64, _dp, f64, _dp, _dp, i64, f64,
                                                      P(vp)])(
                x, self.n, self.d, _c64(y), lam, Uf, _c64(D), self.k, c, C.byref(h)))
            self._destroy = be._fn("problem_destroy", None, [vp])
        else:
            s = _c64(sigma) if self.k else np.zeros(1)
            be._check(be._fn("problem_create", cint, [_dp, i64, i64, _dp, f64, _dp, _dp, i64, cint,
                                                      P(vp)])(
                x, self.n, self.d, _c64(y), lam, Uf, s, self.k, mode, C.byref(h)))
            self._destroy = be._fn("problem_destroy", cint, [vp])
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    @property
    def N(self):
        return self.n + self.d

    def betas(self):
        out = np.empty(self.N)
        self.be._check(self.be._fn("problem_betas", cint, [vp, _dp])(self.h, out))
        return out

    def objective(self, w) -> float:
        out = f64()
        self.be._check(self.be._fn("problem_objective", cint, [vp, _dp, P(f64)])(
            self.h, _c64(w), C.byref(out)))
        return out.value

    def full_gradient(self, w):
        out = np.empty(self.d)
        self.be._check(self.be._fn("problem_full_gradient", cint, [vp, _dp, _dp])(
            self.h, _c64(w), out))
        return out

    def component_gradient(self, i, w):
        out = np.empty(self.d)
        self.be._check(self.be._fn("problem_component_gradient", cint, [vp, i64, _dp, _dp])(
            self.h, i, _c64(w), out))
        return out

    def scalars(self):
        a, b = f64(), f64()
        if self.be.prefix == "skro_":
            m = f64()
            self.be._check(self.be._fn("problem_scalars", cint, [vp, P(f64), P(f64), P(f64)])(
                self.h, C.byref(a), C.byref(b), C.byref(m)))
            return a.value, b.value, m.value
        self.be._check(self.be._fn("problem_scalars", cint, [vp, P(f64), P(f64)])(
            self.h, C.byref(a), C.byref(b)))
        return a.value, b.value, None

    def transformed(self):
        out = np.empty(self.n * self.d)
        self.be._check(self.be._fn("problem_transformed", cint, [vp, _dp])(self.h, out))
        return out.reshape(self.n, self.d)

    def svrg(self, epochs, m, eta, seed, w0=None, reference=float("nan")) -> SvrgOut:
        w0 = np.zeros(self.d) if w0 is None else _c64(w0)
        w = np.empty(self.d)
        tr = np.full(epochs, np.nan)
        done = i64()
        if self.be.prefix == "skro_":
            f = self.be._fn("svrg_solve", cint, [vp, i64, i64, f64, u64, _dp, f64, _dp, _dp, P(i64)])
            rc = f(self.h, epochs, m, eta, seed, w0, reference, w, tr, C.byref(done))
        else:
            f = self.be._fn("svrg_solve", cint, [vp, i64, i64, f64, u64, _dp, f64, _dp, _dp, vp,
                                                 P(i64)])
            rc = f(self.h, epochs, m, eta, seed, w0, reference, w, tr, None, C.byref(done))
        if rc == 5:
            return SvrgOut(w, tr[: done.value], True, self.be._err().decode())
        self.be._check(rc)
        return SvrgOut(w, tr[: done.value])


_port = None
_ref = None


def port() -> _Backend:
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            raise RuntimeError(f"oracle port not built: {PORT_PATH} (run `make -C oracle port`)")
        _port = _Backend(PORT_PATH, "skro_")
    return _port


def ref_available() -> bool:
    try:
        ref()
        return True
    except Exception:
        return False


def ref() -> _Backend:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise RuntimeError(f"reference library not built: {REF_PATH}")
        _ref = _Backend(REF_PATH, "ref_")
    return _ref


def best() -> _Backend:
    """The real reference when it is available, else the restatement."""
    return ref() if ref_available() else port()


# ---------------------------------------------------------------------------
# Synthetic BASELINE instances: host restatement of the DEVICE generator
# (skr_data_generate; oracle/synth.c restates its Philox4x32-10 streams), so the
# CPU reference consumes the instance the GPU generates and times.
def philox4x32_10(ctr, key):
    """Raw Philox4x32-10 block (known-answer tests)."""
    lib = port().lib
    f = lib.skro_philox4x32_10
    u32a = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
    f.restype, f.argtypes = None, [u32a, u32a, u32a]
    out = np.zeros(4, dtype=np.uint32)
    f(np.asarray(ctr, dtype=np.uint32), np.asarray(key, dtype=np.uint32), out)
    return out


def philox_normals(seed: int, stream: int, first: int, count: int, scale: float = 1.0) -> np.ndarray:
    f = port().lib.skro_philox_normals
    f.restype, f.argtypes = None, [u64, C.c_uint32, i64, i64, f64, _dp]
    out = np.empty(count)
    f(seed, stream, first, count, scale, out)
    return out


def synth_haar(cfg) -> np.ndarray:
    """V (d x d): the device draws a d x d Gaussian (stream 2, row-major), QRs its
    column-major view (= its transpose) and fixes signs by sign(diag R)."""
    d = cfg.d
    A = philox_normals(cfg.seed, 2, 0, d * d).reshape(d, d)
    Q, R = np.linalg.qr(A.T)
    return Q * np.sign(np.diag(R))


def synth_instance(cfg, rows: int | None = None, row0: int = 0, V: np.ndarray | None = None,
                   chunk: int = 1 << 16):
    """Rows [row0, row0 + rows) of the config's instance, exactly as the device
    generator lays them out: (X, y) with X (rows, d) float64 or float32 and y
    float64 or float32 (fp32 configs round both).  rows=None: all cfg.n rows.
    The first r rows of the instance at n rows are the instance at r rows."""
    rows = cfg.n - row0 if rows is None else rows
    d = cfg.d
    V = synth_haar(cfg) if V is None else V
    Vt = np.ascontiguousarray(V.T)
    sig = np.ascontiguousarray(cfg.sigma(), dtype=np.float64)
    wstar = philox_normals(cfg.seed, 4, 0, d, 1.0 / math.sqrt(d))
    f32 = cfg.dtype == "f32"
    X = np.empty((rows, d), dtype=np.float32 if f32 else np.float64)
    y = np.empty(rows, dtype=X.dtype)
    g = port().lib.skro_synth_g
    g.restype, g.argtypes = None, [u64, i64, i64, i64, _dp, _dp]
    ts = port().lib.skro_synth_tscale
    ts.restype, ts.argtypes = None, [u64, i64, i64, _dp]
    G = np.empty((min(chunk, max(rows, 1)), d))
    for r in range(0, rows, chunk):
        nr = min(chunk, rows - r)
        Gc = G[:nr]
        g(cfg.seed, row0 + r, nr, d, sig, Gc)
        Xc = Gc @ Vt
        if f32:
            Xc = Xc.astype(np.float32)
        if cfg.t_scale:
            t = np.empty(nr)
            ts(cfg.seed, row0 + r, nr, t)
            Xc = Xc.astype(np.float64) * t[:, None]
            if f32:
                Xc = Xc.astype(np.float32)
        X[r:r + nr] = Xc
        noise = philox_normals(cfg.seed, 5, row0 + r, nr)
        yc = X[r:r + nr].astype(np.float64) @ wstar + cfg.tau * noise
        y[r:r + nr] = yc.astype(np.float32) if f32 else yc
    return X, y


@dataclass
class PipelineOut:
    sigma: np.ndarray
    U: np.ndarray | None
    trace: np.ndarray
    trace_ms: np.ndarray
    w_hat: np.ndarray
    idx: np.ndarray
    alpha: float
    beta_hat: float
    max_row_sq: float
    eta: float
    L_star: float
    L_hat: float
    sketch_ms: float
    precompute_ms: float
    solve_ms: float
    refmin_ms: float
    mode: str
    k_used: int
    full_gradient_ms: float
    rank_reduced: bool


def pipeline(X, y, lam, k, q, seed, epochs, m, eta_rule=0, eta=0.0, mode=2, stop=0.0, idx_count=0,
             want_U=False) -> PipelineOut:
    """The reference's composed pipeline (oracle/ref_capi.cpp ref_pipeline) on ONE
    DataMatrix built from X (n x d, float32 promoted once, or float64)."""
    R = ref()
    f = R._fn("pipeline", cint, [vp, cint, i64, i64, _dp, f64, i64, i64, u64, i64, i64, cint, f64, cint, f64, i64,
                                 _dp, vp, _dp, _dp, P(i64), _dp, vp, _dp])
    X = np.ascontiguousarray(X)
    if X.dtype not in (np.float32, np.float64):
        raise TypeError("X must be float32 or float64")
    n, d = X.shape
    sig = np.zeros(max(k, 1))
    U = np.zeros((d, k), order="F") if (want_U and k > 0) else None
    tr, tms = np.zeros(max(epochs, 1)), np.zeros(max(epochs, 1))
    done = i64(0)
    wh = np.zeros(d)
    idx = np.zeros(max(idx_count, 1), dtype=np.int64)
    sc = np.zeros(16)
    R._check(f(X.ctypes.data, 1 if X.dtype == np.float32 else 0, n, d, _c64(y), lam, k, q, seed, epochs, m, eta_rule,
               eta, mode, stop, idx_count, sig, None if U is None else U.ctypes.data, tr, tms, C.byref(done), wh,
               idx.ctypes.data if idx_count > 0 else None, sc))
    nd = done.value
    return PipelineOut(sig[:int(sc[11])], U, tr[:nd], tms[:nd], wh, idx[:idx_count], sc[0], sc[1], sc[2], sc[3],
                       sc[4], sc[5], sc[6], sc[7], sc[8], sc[9], "dense" if sc[10] == 0 else "lazy", int(sc[11]),
                       sc[12], bool(sc[13]))


def conditioned_matrix(X, lam, U, sigma) -> np.ndarray:
    """The reference's conditioned_matrix(scaled_design, lambda, P) (unguarded)."""
    R = ref()
    f = R._fn("conditioned_matrix", cint, [vp, cint, i64, i64, f64, _dp, _dp, i64, _dp])
    X = np.ascontiguousarray(X)
    n, d = X.shape
    out = np.zeros((d, d))
    k = 0 if U is None else U.shape[1]
    Uc = np.zeros(1) if U is None else np.ascontiguousarray(np.asarray(U).reshape(-1, order="F"))
    sg = np.zeros(1) if sigma is None else _c64(sigma)
    R._check(f(X.ctypes.data, 1 if X.dtype == np.float32 else 0, n, d, lam, Uc, sg, k, out))
    return out
