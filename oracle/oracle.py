"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

Two implementations with one interface:

* ``Ref``  — the unmodified reference library (``/root/reference/proj/core``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libmpnum_ref.so`` with the
  ``ref_shim.cpp`` entry points ("kind": "reference").
* ``Port`` — the C restatement ``oracle/mpnum_oracle.c`` compiled into
  ``oracle/_port/libmpnum_port.so`` ("kind": "port").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg import this module; the product
package never does.

All matrices are column-major float64 numpy arrays holding values that are
representable in the stated precision (0 half, 1 single, 2 double).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmpnum_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libmpnum_port.so")

_i64 = C.c_int64
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="F_CONTIGUOUS")
_vp = C.c_void_p


def build(quiet: bool = True) -> None:
    """Compile the port always, and the reference when its sources exist."""
    targets = ["port"]
    if os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_vp)


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, status: int, info: int = -1):
        super().__init__(f"oracle status {status} (info {info})")
        self.status = status
        self.info = info


class _Base:
    prefix = ""
    kind = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.path = path

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, st: int):
        if st != 0:
            raise OracleError(st, self.last_info())

    def last_info(self) -> int:
        f = self._fn("last_info")
        f.restype = C.c_int
        return f()

    # ---- casts -----------------------------------------------------------
    def encode_f16(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        out = np.empty(x.size, np.uint16)
        self._encode(x, out)
        return out

    def decode_f16(self, b) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.uint16).ravel()
        out = np.empty(b.size, np.float64)
        self._decode(b, out)
        return out

    def convert(self, pin: int, pout: int, raw: np.ndarray) -> np.ndarray:
        """MPArray::converted on raw storage (uint16 / float32 / float64)."""
        raw = np.ascontiguousarray(raw)
        out = np.empty(raw.size, {0: np.uint16, 1: np.float32, 2: np.float64}[pout])
        st = self._fn("convert")(C.c_int(pin), C.c_int(pout), _ptr(raw), _ptr(out),
                                 _i64(raw.size))
        if st is not None and isinstance(st, int):
            self._check(st)
        return out

    # ---- dense kernels ----------------------------------------------------
    def gemm(self, pa, pb, pc, A, B, Cm, ta=False, tb=False, alpha=1.0, beta=0.0):
        A, B, Cm = _f(A), _f(B), _f(Cm).copy(order="F")
        st = self._fn("gemm")(C.c_int(pa), C.c_int(pb), C.c_int(pc),
                              _i64(A.shape[0]), _i64(A.shape[1]), _i64(B.shape[0]),
                              _i64(B.shape[1]), _i64(Cm.shape[0]), _i64(Cm.shape[1]),
                              C.c_int(int(ta)), C.c_int(int(tb)), C.c_double(alpha),
                              C.c_double(beta), _ptr(A), _ptr(B), _ptr(Cm))
        self._check(st)
        return Cm

    def chol(self, p, A):
        A = _f(A)
        out = np.zeros_like(A, order="F")
        self._check(self._chol(p, A, out))
        return out

    def trsm(self, pa, pb, A, B, side_right=False, upper=False, trans=False, alpha=1.0):
        A, B = _f(A), _f(B).copy(order="F")
        self._check(self._trsm(pa, pb, A, B, side_right, upper, trans, alpha))
        return B

    def tile_chol(self, n: int, nb: int, prec: np.ndarray, A) -> np.ndarray:
        """prec: (nt, nt) int array of tile precisions (row i, col j)."""
        A = _f(A)
        prec = np.asfortranarray(prec, dtype=np.int32)
        L = np.zeros_like(A, order="F")
        st = self._fn("tile_chol")(_i64(n), _i64(nb), _ptr(prec), _ptr(A), _ptr(L))
        self._check(st)
        return L

    def rng_uniform(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self._fn("rng_uniform")(C.c_uint64(seed), _i64(n), _ptr(out))
        return out


class Ref(_Base):
    prefix = "ref_"
    kind = "reference"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        self.lib.ref_encode_f16.restype = None
        self.lib.ref_decode_f16.restype = None
        self.lib.ref_rng_uniform.restype = None
        self.lib.ref_rng_normal.restype = None
        self.lib.ref_set_num_threads.restype = None

    def set_num_threads(self, t: int):
        self.lib.ref_set_num_threads(C.c_int(t))

    def _encode(self, x, out):
        self.lib.ref_encode_f16(_ptr(x), _ptr(out), _i64(x.size))

    def _decode(self, b, out):
        self.lib.ref_decode_f16(_ptr(b), _ptr(out), _i64(b.size))

    def _chol(self, p, A, out):
        return self.lib.ref_chol(C.c_int(p), _i64(A.shape[0]), _i64(A.shape[1]), _ptr(A),
                                 _ptr(out))

    def _trsm(self, pa, pb, A, B, side_right, upper, trans, alpha):
        return self.lib.ref_trsm(C.c_int(pa), C.c_int(pb), _i64(A.shape[0]),
                                 _i64(A.shape[1]), _i64(B.shape[0]), _i64(B.shape[1]),
                                 C.c_int(int(side_right)), C.c_int(int(upper)),
                                 C.c_int(int(trans)), C.c_double(alpha), _ptr(A), _ptr(B))

    def crossprod(self, pa, A, pb=None, B=None):
        A = _f(A)
        nb = A.shape[1] if B is None else np.shape(B)[1]
        Bf = None if B is None else _f(B)
        out = np.zeros((A.shape[1], nb), order="F")
        st = self.lib.ref_crossprod(C.c_int(pa), C.c_int(pa if pb is None else pb),
                                    _i64(A.shape[0]), _i64(A.shape[1]),
                                    _i64(A.shape[0] if Bf is None else Bf.shape[0]),
                                    _i64(nb), _ptr(A), _ptr(Bf), _ptr(out))
        self._check(st)
        return out

    def matmul(self, pa, pb, A, B):
        A, B = _f(A), _f(B)
        out = np.zeros((A.shape[0], B.shape[1]), order="F")
        self._check(self.lib.ref_matmul(C.c_int(pa), C.c_int(pb), _i64(A.shape[0]),
                                        _i64(A.shape[1]), _i64(B.shape[0]),
                                        _i64(B.shape[1]), _ptr(A), _ptr(B), _ptr(out)))
        return out

    def solve(self, pa, pb, A, B):
        A, B = _f(A), _f(B)
        out = np.zeros_like(B, order="F")
        self._check(self.lib.ref_solve(C.c_int(pa), C.c_int(pb), _i64(A.shape[0]), _i64(B.shape[1]),
                                       _ptr(A), _ptr(B), _ptr(out)))
        return out

    def chol2inv(self, p, U):
        U = _f(U)
        out = np.zeros_like(U, order="F")
        self._check(self.lib.ref_chol2inv(C.c_int(p), _i64(U.shape[0]), _ptr(U), _ptr(out)))
        return out

    def trisolve(self, upper, pt, pb, T, B):
        T, B = _f(T), _f(B)
        out = np.zeros_like(B, order="F")
        self._check(self.lib.ref_trisolve(C.c_int(int(upper)), C.c_int(pt), C.c_int(pb),
                                          _i64(T.shape[0]), _i64(T.shape[1]),
                                          _i64(B.shape[0]), _i64(B.shape[1]), _ptr(T),
                                          _ptr(B), _ptr(out)))
        return out

    def ew_binary(self, op, pa, pb, A, B):
        A, B = _f(A), _f(B)
        out = np.zeros_like(A, order="F")
        self._check(self.lib.ref_ew_binary(C.c_int(op), C.c_int(pa), C.c_int(pb),
                                           _i64(A.shape[0]), _i64(A.shape[1]),
                                           _i64(B.shape[0]), _i64(B.shape[1]), _ptr(A),
                                           _ptr(B), _ptr(out)))
        return out

    def ew_scalar(self, op, p, A, s):
        A = _f(A)
        out = np.zeros_like(A, order="F")
        self._check(self.lib.ref_ew_scalar(C.c_int(op), C.c_int(p), _i64(A.shape[0]),
                                           _i64(A.shape[1]), _ptr(A), C.c_double(s),
                                           _ptr(out)))
        return out

    def ew_unary(self, op, p, A):
        A = _f(A)
        out = np.zeros_like(A, order="F")
        self._check(self.lib.ref_ew_unary(C.c_int(op), C.c_int(p), _i64(A.shape[0]),
                                          _i64(A.shape[1]), _ptr(A), _ptr(out)))
        return out

    def reduce(self, op, p, A) -> float:
        A = _f(A)
        r = C.c_double()
        self._check(self.lib.ref_reduce(C.c_int(op), C.c_int(p), _i64(A.shape[0]),
                                        _i64(A.shape[1]), _ptr(A), C.byref(r)))
        return r.value

    def transpose(self, p, A):
        A = _f(A)
        out = np.zeros((A.shape[1], A.shape[0]), order="F")
        self._check(self.lib.ref_transpose(C.c_int(p), _i64(A.shape[0]), _i64(A.shape[1]),
                                           _ptr(A), _ptr(out)))
        return out

    def diag(self, p, A):
        A = _f(A)
        out = np.zeros(min(A.shape), np.float64)
        self._check(self.lib.ref_diag(C.c_int(p), _i64(A.shape[0]), _i64(A.shape[1]),
                                      _ptr(A), _ptr(out)))
        return out

    def rng_normal(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.ref_rng_normal(C.c_uint64(seed), _i64(n), _ptr(out))
        return out

    def grid_matern(self, side, n, nu=0.5, rng=1.0, sigma2=1.0, prec=2):
        out = np.zeros((n, n), order="F")
        self._check(self.lib.ref_grid_matern(_i64(side), _i64(n), C.c_double(nu),
                                             C.c_double(rng), C.c_double(sigma2),
                                             C.c_int(prec), _ptr(out)))
        return out

    def gaussian_nll(self, prec, z, cov) -> float:
        z, cov = _f(z).ravel(), _f(cov)
        r = C.c_double()
        self._check(self.lib.ref_gaussian_nll(C.c_int(prec), _i64(z.size), _ptr(z),
                                              _ptr(cov), C.byref(r)))
        return r.value

    def sample_gp(self, cov, seed: int) -> np.ndarray:
        cov = _f(cov)
        out = np.zeros(cov.shape[0], np.float64)
        self._check(self.lib.ref_sample_gp(_i64(cov.shape[0]), _ptr(cov),
                                           C.c_uint64(seed), _ptr(out)))
        return out

    def matern_mle(self, prec, side, z, init_log_range, init_log_sigma2, max_iter=200, tol=1e-4):
        """matern_mle (workloads.cpp:89-110) on the first len(z) points of the side x side grid."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = [C.c_double(), C.c_double(), C.c_double(), C.c_int()]
        self._check(self.lib.ref_matern_mle(C.c_int(prec), _i64(side), _i64(z.size), _ptr(z),
                                            C.c_double(init_log_range), C.c_double(init_log_sigma2),
                                            C.c_int(max_iter), C.c_double(tol), C.byref(out[0]),
                                            C.byref(out[1]), C.byref(out[2]), C.byref(out[3])))
        return {"range": out[0].value, "sigma2": out[1].value, "nll": out[2].value,
                "iterations": out[3].value}

    def tile_gemm(self, A, ptA, nbA, B, ptB, nbB, Cm, ptC, nbC, ta=False, tb=False,
                  alpha=1.0, beta=0.0):
        """nbX = (rows_per_tile, cols_per_tile); ptX = tile-precision grid."""
        A, B, Cm = _f(A), _f(B), _f(Cm).copy(order="F")
        ptA, ptB, ptC = (np.asfortranarray(p, dtype=np.int32) for p in (ptA, ptB, ptC))
        st = self.lib.ref_tile_gemm(
            _i64(A.shape[0]), _i64(A.shape[1]), _i64(nbA[0]), _i64(nbA[1]), _ptr(ptA), _ptr(A),
            _i64(B.shape[0]), _i64(B.shape[1]), _i64(nbB[0]), _i64(nbB[1]), _ptr(ptB), _ptr(B),
            _i64(Cm.shape[0]), _i64(Cm.shape[1]), _i64(nbC[0]), _i64(nbC[1]), _ptr(ptC),
            _ptr(Cm), C.c_int(int(ta)), C.c_int(int(tb)), C.c_double(alpha),
            C.c_double(beta))
        self._check(st)
        return Cm

    def tile_trsm(self, A, ptA, nb, B, ptB, nbB, side_right=False, upper=False,
                  trans=False, alpha=1.0):
        A, B = _f(A), _f(B).copy(order="F")
        ptA, ptB = (np.asfortranarray(p, dtype=np.int32) for p in (ptA, ptB))
        st = self.lib.ref_tile_trsm(_i64(A.shape[0]), _i64(nb), _ptr(ptA), _ptr(A),
                                    _i64(B.shape[0]), _i64(B.shape[1]), _i64(nbB[0]),
                                    _i64(nbB[1]), _ptr(ptB), _ptr(B), C.c_int(int(side_right)),
                                    C.c_int(int(upper)), C.c_int(int(trans)),
                                    C.c_double(alpha))
        self._check(st)
        return B


class Port(_Base):
    prefix = "mpo_"
    kind = "port"

    def __init__(self, path: str = PORT_SO):
        super().__init__(path)
        self.lib.mpo_encode_f16.restype = C.c_uint16
        self.lib.mpo_encode_f16.argtypes = [C.c_double]
        self.lib.mpo_decode_f16.restype = C.c_double
        self.lib.mpo_decode_f16.argtypes = [C.c_uint16]
        self.lib.mpo_convert.restype = None
        self.lib.mpo_rng_uniform.restype = None
        self.lib.mpo_reduce.restype = C.c_double
        self.lib.mpo_logdet_lower.restype = C.c_double

    def _encode(self, x, out):
        for i, v in enumerate(x):
            out[i] = self.lib.mpo_encode_f16(float(v))

    def _decode(self, b, out):
        for i, v in enumerate(b):
            out[i] = self.lib.mpo_decode_f16(int(v))

    def _chol(self, p, A, out):
        if A.shape[0] != A.shape[1]:
            return 1
        return self.lib.mpo_chol(C.c_int(p), _i64(A.shape[0]), _ptr(A), _ptr(out))

    def _trsm(self, pa, pb, A, B, side_right, upper, trans, alpha):
        return self.lib.mpo_trsm(C.c_int(pa), C.c_int(pb), _i64(A.shape[0]),
                                 _i64(B.shape[0]), _i64(B.shape[1]), C.c_int(int(side_right)),
                                 C.c_int(int(upper)), C.c_int(int(trans)), C.c_double(alpha),
                                 _ptr(A), _ptr(B))

    def crossprod(self, pa, A, pb=None, B=None):
        A = _f(A)
        Bf = None if B is None else _f(B)
        nb = A.shape[1] if B is None else Bf.shape[1]
        out = np.zeros((A.shape[1], nb), order="F")
        self._check(self.lib.mpo_crossprod(C.c_int(pa), C.c_int(pa if pb is None else pb),
                                           _i64(A.shape[0]), _i64(A.shape[1]),
                                           _i64(A.shape[0] if Bf is None else Bf.shape[0]),
                                           _i64(nb), _ptr(A), _ptr(Bf), _ptr(out)))
        return out

    def ew_binary(self, op, pa, pb, A, B):
        A, B = _f(A), _f(B)
        out = np.zeros_like(A, order="F")
        self.lib.mpo_ew_binary(C.c_int(op), C.c_int(pa), C.c_int(pb), _i64(A.size),
                               _ptr(A), _ptr(B), _ptr(out))
        return out

    def ew_scalar(self, op, p, A, s):
        A = _f(A)
        out = np.zeros_like(A, order="F")
        self.lib.mpo_ew_scalar(C.c_int(op), C.c_int(p), _i64(A.size), _ptr(A),
                               C.c_double(s), _ptr(out))
        return out

    def reduce(self, op, p, A) -> float:
        A = _f(A)
        return self.lib.mpo_reduce(C.c_int(op), _i64(A.size), _ptr(A))

    def logdet_lower(self, L) -> float:
        L = _f(L)
        return self.lib.mpo_logdet_lower(_i64(L.shape[0]), _ptr(L))


def round_to(x, p: int) -> np.ndarray:
    """round_to_precision (precision.cpp:111-120), vectorised with numpy.

    numpy's float64->float16 cast is round-to-nearest-even straight from
    double, the same rounding as encode_f16; NaN payloads never matter here
    because decode maps every half NaN to the canonical quiet NaN.
    """
    x = np.asarray(x, dtype=np.float64)
    if p == 0:
        return x.astype(np.float16).astype(np.float64)
    if p == 1:
        return x.astype(np.float32).astype(np.float64)
    return x.copy()


def best() -> _Base:
    """The reference when it was built, else the C port."""
    return Ref() if os.path.exists(REF_SO) else Port()
