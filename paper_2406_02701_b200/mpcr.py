"""Host-side mirror of the reference API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ core
(``mpnum``: precision.hpp, array.hpp, linalg.hpp) and the paper's MPCRTile
API, so callers and parity tests read like the reference's
own tests.  All storage is device-resident; numpy arrays cross the boundary
only in ``from_numpy`` / ``to_numpy``.
"""
from __future__ import annotations

import ctypes as C
import enum
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import MPError, check, lib


class Precision(enum.IntEnum):  # precision.hpp:11
    Half = 0
    Single = 1
    Double = 2


class BinaryOp(enum.IntEnum):  # array.hpp:94
    Add = 0
    Sub = 1
    Mul = 2
    Div = 3


class UnaryOp(enum.IntEnum):  # array.hpp:95
    Log = 0
    Exp = 1
    Sqrt = 2
    Abs = 3


class ReduceOp(enum.IntEnum):  # array.hpp:96
    Sum = 0
    SquareSum = 1
    Min = 2
    Max = 3
    Mean = 4


class Side(enum.IntEnum):  # linalg.hpp:21
    Left = 0
    Right = 1


NP_STORAGE = {Precision.Half: np.uint16, Precision.Single: np.float32,
              Precision.Double: np.float64}
UNIT_ROUNDOFF = {Precision.Half: 2.0 ** -11, Precision.Single: 2.0 ** -24,
                 Precision.Double: 2.0 ** -53}  # precision.cpp:11-15


def promote(a: Precision, b: Precision) -> Precision:  # precision.hpp:31-33
    return Precision(max(int(a), int(b)))


def parse_precision(name: str) -> Precision:  # precision.cpp:36-42
    table = {"half": Precision.Half, "single": Precision.Single, "double": Precision.Double}
    if name not in table:
        raise MPError(11, f'unknown precision: "{name}" (expected half, single, or double)')
    return table[name]


class Context:
    """Device, streams and workspace (mp_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().mp_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            lib().mp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        check(lib().mp_ctx_synchronize(self.h))

    def set_stream(self, stream_ptr: int):
        check(lib().mp_ctx_set_stream(self.h, C.c_void_p(stream_ptr)))

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib().mp_ctx_get_stream(self.h, C.byref(s)))
        return s.value or 0

    def prof_enable(self, on: bool = True):
        check(lib().mp_prof_enable(self.h, int(on)))

    def prof_reset(self):
        check(lib().mp_prof_reset(self.h))

    def prof_trace(self, enable: bool = True):
        """Record a per-launch timeline (needs prof_enable)."""
        check(lib().mp_prof_trace(self.h, int(enable)))

    def prof_trace_dump(self, path: str):
        check(lib().mp_prof_trace_dump(self.h, path.encode()))

    def prof_query(self, cls: int):
        ms, n, w = C.c_double(), C.c_int64(), C.c_double()
        check(lib().mp_prof_query(self.h, cls, C.byref(ms), C.byref(n), C.byref(w)))
        return ms.value, n.value, w.value

    def prof_digit_products(self):
        """(INT8 digit-pair MMAs issued, FP64 output tiles) of the Ozaki kernel
        since the last prof_reset (profiling runs only)."""
        a, b = C.c_int64(), C.c_int64()
        check(lib().mp_prof_digit_products(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def launch_count(self) -> int:
        n = C.c_int64()
        check(lib().mp_launch_count(self.h, C.byref(n)))
        return n.value


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


class MPArray:
    """Device MPArray (array.hpp:18-82): column-major, precision-tagged."""

    def __init__(self, handle, ctx: Context, owner: bool = True):
        self.h = handle
        self.ctx = ctx
        self._owner = owner

    # ---- construction (array.hpp:23-41) ------------------------------------
    @classmethod
    def zeros(cls, size: int, prec: Precision, ctx: Context | None = None) -> "MPArray":
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().mp_array_create(ctx.h, int(prec), size, 1, 0, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def zeros_matrix(cls, rows: int, cols: int, prec: Precision,
                     ctx: Context | None = None) -> "MPArray":
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib().mp_array_create(ctx.h, int(prec), rows, cols, 1, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_doubles(cls, values, rows: int, cols: int, prec: Precision,
                     ctx: Context | None = None) -> "MPArray":
        """Column-major values rounded to prec (array.cpp:66-76)."""
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).ravel())
        if v.size != rows * cols:
            raise MPError(1, f"from_doubles: {v.size} values cannot fill a {rows}x{cols} matrix")
        a = cls.zeros_matrix(rows, cols, prec, ctx)
        check(lib().mp_array_from_doubles(a.h, v.ctypes.data_as(C.c_void_p), v.size))
        return a

    @classmethod
    def from_numpy(cls, m: np.ndarray, prec: Precision, ctx: Context | None = None) -> "MPArray":
        m = np.asarray(m, dtype=np.float64)
        if m.ndim == 1:
            m = m.reshape(-1, 1)
        return cls.from_doubles(np.asfortranarray(m).ravel(order="F"), m.shape[0], m.shape[1],
                                prec, ctx)

    @classmethod
    def from_storage(cls, raw: np.ndarray, rows: int, cols: int, prec: Precision,
                     ctx: Context | None = None) -> "MPArray":
        """Upload raw storage bytes (uint16 / float32 / float64), column-major."""
        a = cls.zeros_matrix(rows, cols, prec, ctx)
        r = np.ascontiguousarray(raw, dtype=NP_STORAGE[prec]).ravel(order="F")
        check(lib().mp_array_upload(a.h, r.ctypes.data_as(C.c_void_p), r.nbytes))
        return a

    def close(self):
        if self.h and self._owner:
            lib().mp_array_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- info ----------------------------------------------------------------
    def _info(self):
        p, r, c, ld, im, ptr = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int(), C.c_void_p()
        check(lib().mp_array_info(self.h, C.byref(p), C.byref(r), C.byref(c), C.byref(ld),
                                  C.byref(im), C.byref(ptr)))
        return Precision(p.value), r.value, c.value, ld.value, bool(im.value), ptr.value

    def precision(self) -> Precision:
        return self._info()[0]

    def rows(self) -> int:
        return self._info()[1]

    def cols(self) -> int:
        return self._info()[2]

    def size(self) -> int:
        _, r, c, *_ = self._info()
        return r * c

    def is_matrix(self) -> bool:
        return self._info()[4]

    def data_ptr(self) -> int:
        return self._info()[5]

    def to_matrix(self, rows: int, cols: int):
        check(lib().mp_array_to_matrix(self.h, rows, cols))

    # ---- element access (array.hpp:52-62) ----------------------------------
    def get(self, i: int, j: int = 0) -> float:
        v = C.c_double()
        check(lib().mp_array_get(self.h, i, j, C.byref(v)))
        return v.value

    def set(self, i: int, j: int, v: float):
        check(lib().mp_array_set(self.h, i, j, float(v)))

    def to_doubles(self) -> np.ndarray:
        out = np.empty(self.size(), np.float64)
        check(lib().mp_array_to_doubles(self.h, out.ctypes.data_as(C.c_void_p), out.size))
        return out

    def to_numpy(self) -> np.ndarray:
        _, r, c, *_ = self._info()
        return self.to_doubles().reshape((r, c), order="F")

    def storage(self) -> np.ndarray:
        """Raw storage bytes as uint16 / float32 / float64, column-major."""
        p, r, c, *_ = self._info()
        out = np.empty(r * c, NP_STORAGE[p])
        check(lib().mp_array_download(self.h, out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def half_bits(self, i: int) -> int:  # array.hpp:67
        if self.precision() != Precision.Half:
            raise MPError(11, "half_bits: array is not half precision")
        return int(self.storage()[i])

    # ---- MPArray::converted (array.cpp:187-191) ----------------------------
    def converted(self, prec: Precision) -> "MPArray":
        _, r, c, _, im, _ = self._info()
        out = MPArray.zeros_matrix(r, c, prec, self.ctx) if im else MPArray.zeros(r, prec, self.ctx)
        check(lib().mp_convert(self.ctx.h, self.h, out.h))
        return out


def _like(a: MPArray, prec: Precision, rows=None, cols=None) -> MPArray:
    _, r, c, _, im, _ = a._info()
    r = r if rows is None else rows
    c = c if cols is None else cols
    if im or cols is not None:
        return MPArray.zeros_matrix(r, c, prec, a.ctx)
    return MPArray.zeros(r, prec, a.ctx)


# ---- elementwise (array.hpp:84-106) ---------------------------------------
def ew_binary(op: BinaryOp, a: MPArray, b: MPArray) -> MPArray:
    if a.rows() != b.rows() or a.cols() != b.cols() or a.is_matrix() != b.is_matrix():
        raise MPError(1, "ew_binary: shapes do not match")
    out = _like(a, promote(a.precision(), b.precision()))
    check(lib().mp_ew_binary(a.ctx.h, int(op), a.h, b.h, out.h))
    return out


def ew_scalar(op: BinaryOp, a: MPArray, s: float) -> MPArray:
    out = _like(a, a.precision())
    check(lib().mp_ew_scalar(a.ctx.h, int(op), a.h, float(s), out.h))
    return out


def ew_unary(op: UnaryOp, a: MPArray) -> MPArray:
    out = _like(a, a.precision())
    check(lib().mp_ew_unary(a.ctx.h, int(op), a.h, out.h))
    return out


def reduce(op: ReduceOp, a: MPArray) -> float:
    v = C.c_double()
    check(lib().mp_reduce(a.ctx.h, int(op), a.h, C.byref(v)))
    return v.value


def transpose(a: MPArray) -> MPArray:
    if not a.is_matrix():
        raise MPError(3, "transpose: input is not a matrix")
    out = MPArray.zeros_matrix(a.cols(), a.rows(), a.precision(), a.ctx)
    check(lib().mp_transpose(a.ctx.h, a.h, out.h))
    return out


def diag(a: MPArray) -> MPArray:
    if not a.is_matrix():
        raise MPError(3, "diag: input is not a matrix")
    out = MPArray.zeros(max(1, min(a.rows(), a.cols())), a.precision(), a.ctx)
    check(lib().mp_diag(a.ctx.h, a.h, out.h))
    return out


class linalg:
    """linalg.hpp:23-54 on the device."""

    @staticmethod
    def gemm(a: MPArray, b: MPArray, c: MPArray, trans_a=False, trans_b=False, alpha=1.0,
             beta=0.0) -> None:
        check(lib().mp_gemm(a.ctx.h, a.h, b.h, c.h, int(trans_a), int(trans_b), float(alpha),
                            float(beta)))

    @staticmethod
    def matmul(a: MPArray, b: MPArray) -> MPArray:
        if not a.is_matrix() or not b.is_matrix():
            raise MPError(3, "matmul: input is not a matrix")
        out = MPArray.zeros_matrix(a.rows(), b.cols(), promote(a.precision(), b.precision()),
                                   a.ctx)
        check(lib().mp_matmul(a.ctx.h, a.h, b.h, out.h))
        return out

    @staticmethod
    def crossprod(a: MPArray, b: MPArray | None = None) -> MPArray:
        if not a.is_matrix() or (b is not None and not b.is_matrix()):
            raise MPError(3, "crossprod: input is not a matrix")
        bb = a if b is None else b
        out = MPArray.zeros_matrix(a.cols(), bb.cols(), promote(a.precision(), bb.precision()),
                                   a.ctx)
        check(lib().mp_crossprod(a.ctx.h, a.h, None if b is None else b.h, out.h))
        return out

    @staticmethod
    def chol(a: MPArray) -> MPArray:
        out = MPArray.zeros_matrix(a.rows(), a.cols(), a.precision(), a.ctx)
        info = C.c_int64(-1)
        check(lib().mp_chol(a.ctx.h, a.h, out.h, C.byref(info)), info.value)
        return out

    @staticmethod
    def trsm(a: MPArray, b: MPArray, side: Side, upper: bool, trans: bool, alpha: float) -> None:
        check(lib().mp_trsm(a.ctx.h, a.h, b.h, int(side), int(upper), int(trans), float(alpha)))

    @staticmethod
    def forwardsolve(l: MPArray, b: MPArray) -> MPArray:
        out = _like(b, promote(l.precision(), b.precision()))
        check(lib().mp_forwardsolve(l.ctx.h, l.h, b.h, out.h))
        return out

    @staticmethod
    def backsolve(u: MPArray, b: MPArray) -> MPArray:
        out = _like(b, promote(u.precision(), b.precision()))
        check(lib().mp_backsolve(u.ctx.h, u.h, b.h, out.h))
        return out

    @staticmethod
    def solve(a: MPArray, b: MPArray | None = None) -> MPArray:
        """solve(a[, b]) (linalg.cpp:544-575); without b, the inverse."""
        if b is None:
            b = MPArray.from_numpy(np.eye(a.rows()), a.precision(), a.ctx)
        out = _like(b, promote(a.precision(), b.precision()))
        check(lib().mp_solve(a.ctx.h, a.h, b.h, out.h))
        return out

    @staticmethod
    def chol2inv(u: MPArray) -> MPArray:
        """chol2inv (linalg.cpp:481-488): (U^T U)^-1 from the upper factor."""
        out = MPArray.zeros_matrix(u.rows(), u.cols(), u.precision(), u.ctx)
        check(lib().mp_chol2inv(u.ctx.h, u.h, out.h))
        return out


def rng_uniform(seed: int, n: int, skip: int = 0) -> np.ndarray:
    """n uniforms of the reference Rng(seed) (rng.cpp:9-36) after `skip` draws."""
    out = np.empty(n, np.float64)
    check(lib().mp_rng_uniform(seed, skip, n, out.ctypes.data_as(C.c_void_p)))
    return out


def rng_normal(seed: int, n: int) -> np.ndarray:
    """n standard normals of the reference Rng(seed) (rng.cpp:38-50)."""
    out = np.empty(n, np.float64)
    check(lib().mp_rng_normal(seed, n, out.ctypes.data_as(C.c_void_p)))
    return out


def random_uniform_matrix(rows: int, cols: int, rng_seed: int, skip: int = 0) -> np.ndarray:
    """acceptance.cpp:30-36 random_uniform: column-major fill from Rng(seed)."""
    return rng_uniform(rng_seed, rows * cols, skip).reshape((rows, cols), order="F")


class KernelKey(C.Structure):
    """dispatch::KernelKey (dispatch.hpp): input precisions, promoted output;
    in_b = -1 for unary operations."""
    _fields_ = [("in_a", C.c_int), ("in_b", C.c_int), ("out", C.c_int)]

    def __repr__(self):
        b = None if self.in_b < 0 else Precision(self.in_b)
        return f"KernelKey(in_a={Precision(self.in_a)!r}, in_b={b!r}, out={Precision(self.out)!r})"


class dispatch:
    """mpnum::dispatch (dispatch.cpp:46-137): the op-name registry on device arrays."""

    @staticmethod
    def is_unary(op: str) -> bool:
        u = C.c_int()
        check(lib().mp_op_is_unary(op.encode(), C.byref(u)))
        return bool(u.value)

    @staticmethod
    def resolve(op: str, a: Precision, b: Precision | None = None) -> KernelKey:
        k = KernelKey()
        check(lib().mp_resolve(op.encode(), int(a), -1 if b is None else int(b), C.byref(k)))
        return k

    @staticmethod
    def execute(key: KernelKey, op: str, a: MPArray, b: MPArray | None = None) -> MPArray:
        out = C.c_void_p()
        check(lib().mp_execute(a.ctx.h, C.byref(key), op.encode(), a.h, b.h if b is not None else None,
                               C.byref(out)))
        return MPArray(out, a.ctx)


class MPCRTile:
    """MPCRTile: per-tile precisions, tiles on the device.

    ``precisions`` is a (tiles_r, tiles_c) grid of Precision / ints / the
    strings "half" | "single" | "double", like R's precision matrix.
    """

    def __init__(self, rows: int, cols: int, rows_per_tile: int, cols_per_tile: int,
                 values=None, precisions=None, ctx: Context | None = None, _handle=None,
                 grid: "ProcessGrid | None" = None):
        self.ctx = ctx or (grid.ctx if grid is not None else default_context())
        self.grid = grid
        if _handle is not None:
            self.h = _handle
        else:
            tr, tc = rows // max(rows_per_tile, 1), cols // max(cols_per_tile, 1)
            if precisions is None:
                precisions = np.full((tr, tc), int(Precision.Double))
            pg = np.array([[int(parse_precision(p)) if isinstance(p, str) else int(p)
                            for p in row] for row in np.atleast_2d(np.asarray(precisions,
                                                                              dtype=object))])
            pcol = np.asfortranarray(pg, dtype=np.int32).ravel(order="F")
            h = C.c_void_p()
            if grid is not None:
                if rows != cols or rows_per_tile != cols_per_tile:
                    raise ValueError("distributed MPCRTile: square matrix with square tiles")
                check(lib().mp_tile_create_dist(self.ctx.h, grid.h, rows, rows_per_tile,
                                                pcol.ctypes.data_as(C.POINTER(C.c_int)), C.byref(h)))
            else:
                check(lib().mp_tile_create(self.ctx.h, rows, cols, rows_per_tile, cols_per_tile,
                                           pcol.ctypes.data_as(C.POINTER(C.c_int)), C.byref(h)))
            self.h = h
            if values is not None:
                self.set_values(values)

    def close(self):
        if self.h:
            lib().mp_tile_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        v = [C.c_int64() for _ in range(6)]
        check(lib().mp_tile_info(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def set_values(self, values):
        rows, cols, *_ = self.info()
        m = np.asfortranarray(np.asarray(values, dtype=np.float64).reshape((rows, cols), order="F"))
        check(lib().mp_tile_set_values(self.h, m.ctypes.data_as(C.c_void_p)))

    def to_numpy(self) -> np.ndarray:
        rows, cols, *_ = self.info()
        out = np.empty((rows, cols), order="F")
        check(lib().mp_tile_get_values(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def get_rows(self, rows) -> np.ndarray:
        """Selected rows (0-based) of the whole matrix as doubles, shape
        (len(rows), cols); tiles stored on other ranks read as zeros."""
        _, cols, *_ = self.info()
        r = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((r.size, cols))
        check(lib().mp_tile_get_rows(self.h, r.ctypes.data_as(C.c_void_p), r.size,
                                     out.ctypes.data_as(C.c_void_p)))
        return out

    def owns(self, i: int, j: int) -> bool:
        """True if tile (i, j) (0-based) is stored by this rank."""
        return bool(lib().mp_tile_owns(self.h, i, j))

    def GetTile(self, rowidx: int, colidx: int) -> MPArray:
        """MPCRTile.GetTile: 1-based, a view of the tile."""
        v = C.c_void_p()
        check(lib().mp_tile_get_tile(self.h, rowidx - 1, colidx - 1, C.byref(v)))
        return MPArray(v, self.ctx, owner=True)

    def tile_precision(self, i: int, j: int) -> Precision:
        p = C.c_int()
        check(lib().mp_tile_precision(self.h, i, j, C.byref(p)))
        return Precision(p.value)

    def fill_matern(self, grid_side: int, nu=0.5, range_=0.1, variance=1.0):
        check(lib().mp_tile_fill_matern(self.ctx.h, self.h, grid_side, nu, range_, variance))

    def fill_matern_points(self, x: np.ndarray, y: np.ndarray, nu=0.5, range_=0.1,
                           variance=1.0, nugget=0.0):
        """Matern covariance of host locations (x, y), generated on the device."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        check(lib().mp_tile_fill_matern_points(self.ctx.h, self.h, x.ctypes.data_as(C.c_void_p),
                                               y.ctypes.data_as(C.c_void_p), x.size, nu, range_,
                                               variance, nugget))

    def convert_from(self, src: "MPCRTile"):
        """Every tile of src converted into this tile object's precision for it."""
        check(lib().mp_tile_convert(self.ctx.h, self.h, src.h))

    def copy_from(self, src: "MPCRTile"):
        check(lib().mp_tile_copy(self.ctx.h, self.h, src.h))

    def logdet(self) -> float:
        v = C.c_double()
        check(lib().mp_tile_logdet(self.ctx.h, self.h, C.byref(v)))
        return v.value


def tile_gemm(a: MPCRTile, b: MPCRTile, c: MPCRTile, transpose_a=False, transpose_b=False,
              alpha=1.0, beta=0.0, num_threads: int = 1) -> None:
    """MPCRTile.gemm; num_threads is accepted and ignored."""
    check(lib().mp_tile_gemm(a.ctx.h, a.h, b.h, c.h, int(transpose_a), int(transpose_b),
                             float(alpha), float(beta)))


def tile_chol(x: MPCRTile, overwrite_input: bool = True, num_threads: int = 1) -> MPCRTile:
    """chol(MPCRTile): lower L."""
    out = C.c_void_p()
    info = C.c_int64(-1)
    check(lib().mp_tile_chol(x.ctx.h, x.h, int(overwrite_input), C.byref(out), C.byref(info)),
          info.value)
    if overwrite_input:
        return x
    return MPCRTile(0, 0, 0, 0, ctx=x.ctx, _handle=out)


def gaussian_nll(z, cov: MPCRTile, jitter: float = 1e-6, max_jitter: float = 1e-3) -> dict:
    """gaussian_nll (workloads.cpp:74-87) on a mixed-precision MPCRTile; `cov`
    is factored in place.  jitter <= 0 disables chol_with_jitter (the
    reference uses 1e-6 .. 1e-3 whenever the factor is not all-double)."""
    z = np.ascontiguousarray(np.asarray(z, dtype=np.float64).ravel())
    out = [C.c_double() for _ in range(4)]
    check(lib().mp_tile_gaussian_nll(cov.ctx.h, cov.h, z.ctypes.data_as(C.c_void_p),
                                     float(jitter), float(max_jitter),
                                     *[C.byref(o) for o in out]))
    return dict(zip(("nll", "logdet", "quad", "jitter"), (o.value for o in out)))


def matern_mle(cov: MPCRTile, x, y, z, init_log_range: float, init_log_sigma2: float, nu: float = 0.5,
               max_iter: int = 200, tol: float = 1e-4, jitter: float = 1e-6,
               max_jitter: float = 1e-3) -> dict:
    """matern_mle (workloads.cpp:89-110): Nelder-Mead over (log range,
    log sigma2) with every likelihood evaluated on the GPU in `cov`."""
    n = cov.info()[0]
    xs, ys, zs = (np.ascontiguousarray(np.asarray(v, dtype=np.float64).ravel()) for v in (x, y, z))
    if not (xs.size == ys.size == zs.size == n):
        raise MPError(1, "matern_mle: x, y and z must have n entries")
    out = [C.c_double(), C.c_double(), C.c_double(), C.c_int(), C.c_int()]
    check(lib().mp_tile_matern_mle(cov.ctx.h, cov.h, xs.ctypes.data_as(C.c_void_p),
                                   ys.ctypes.data_as(C.c_void_p), zs.ctypes.data_as(C.c_void_p), n,
                                   float(nu), float(init_log_range), float(init_log_sigma2), int(max_iter),
                                   float(tol), float(jitter), float(max_jitter), *[C.byref(o) for o in out]))
    return {"range": out[0].value, "sigma2": out[1].value, "nll": out[2].value,
            "iterations": out[3].value, "converged": bool(out[4].value)}


def tile_trsm(a: MPCRTile, b: MPCRTile, side: str = "L", upper_triangle: bool = False,
              transpose: bool = False, alpha: float = 1.0) -> None:
    """MPCRTile.trsm: b overwritten with X."""
    s = {"L": Side.Left, "R": Side.Right}[side]
    check(lib().mp_tile_trsm(a.ctx.h, a.h, b.h, int(s), int(upper_triangle), int(transpose),
                             float(alpha)))


# ---- multi-GPU: 2D block-cyclic process grid -----------------

DIST_OPS = {1: "potrf", 2: "bcast_diag", 3: "trsm", 4: "bcast_panel", 5: "update"}


def dist_owner(i: int, j: int, P: int, Q: int) -> int:
    """Rank holding tile (i, j) of a P x Q block-cyclic grid."""
    return int(lib().mp_dist_owner(i, j, P, Q))


def dist_schedule(rank: int, P: int, Q: int, tiles: int, precisions=None) -> np.ndarray:
    """The rank's action list of the distributed tiled Cholesky, as an
    (count, 7) int32 array of (op, k, i, j, root, precision, comm) rows (comm
    0 world, 1 process row, 2 process column) — the same plan the GPU
    executor runs (csrc/dist.cpp)."""
    if precisions is None:
        precisions = np.full((tiles, tiles), 2)
    pcol = np.asfortranarray(np.asarray(precisions, dtype=np.int32)).ravel(order="F")
    cnt = C.c_int64()
    pp = pcol.ctypes.data_as(C.POINTER(C.c_int))
    check(lib().mp_dist_schedule(rank, P, Q, tiles, pp, None, 0, C.byref(cnt)))
    out = np.zeros((cnt.value, 7), dtype=np.int32)
    check(lib().mp_dist_schedule(rank, P, Q, tiles, pp, out.ctypes.data_as(C.POINTER(C.c_int32)),
                                 cnt.value, C.byref(cnt)))
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().mp_nccl_unique_id(buf))
    return buf.raw


class ProcessGrid:
    """P x Q process grid over NCCL (one process per GPU).  Rank 0 makes the
    id with ``nccl_unique_id()`` and shares it (e.g. torch.distributed
    broadcast_object_list); world == 1 needs none."""

    def __init__(self, rank: int, world: int, P: int, Q: int, uid: bytes | None = None,
                 ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.rank, self.world, self.P, self.Q = rank, world, P, Q
        h = C.c_void_p()
        check(lib().mp_dist_create(self.ctx.h, rank, world, P, Q, uid, C.byref(h)))
        self.h = h

    def owner(self, i: int, j: int) -> int:
        return dist_owner(i, j, self.P, self.Q)

    @classmethod
    def simulated(cls, ctxs, P: int, Q: int) -> list:
        """P x Q ranks on ONE GPU (test harness, mp_dist_create_sim): one grid
        handle per rank, rank r on ctxs[r]; run the ranks' calls concurrently
        from one thread each."""
        world = P * Q
        arr = (C.c_void_p * world)(*[c.h for c in ctxs])
        hs = (C.c_void_p * world)()
        check(lib().mp_dist_create_sim(arr, world, P, Q, hs))
        out = []
        for r in range(world):
            g = cls.__new__(cls)
            g.ctx, g.rank, g.world, g.P, g.Q = ctxs[r], r, world, P, Q
            g.h = C.c_void_p(hs[r])
            out.append(g)
        return out

    def close(self):
        if self.h:
            lib().mp_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
