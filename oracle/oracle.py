"""numpy bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/librc_oracle.so`` (the C restatement, rc_oracle.c) and, when present,
``oracle/_ref/librc_ref.so`` (the unmodified reference headers compiled in place by
oracle/Makefile).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module; the product
package ``paper_2512_08888_b200`` never does (tests/test_boundary.py checks that).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "librc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librc_ref.so")

GROUPS = {"single": 0, "p4": 1, "p4m": 2, "steer": 3}
POOLS = {"none": 0, "avg": 1, "max": 2, "subgroup": 3}
CONVENTIONS = {"scatter": 0, "raw": 1}


class _Desc(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "n", "c_in", "h", "w", "c_out", "k", "group", "orientations", "pool",
        "pool_group", "convention")]


@dataclass
class Desc:
    n: int
    c_in: int
    h: int
    w: int
    c_out: int
    k: int = 3
    group: str = "single"
    orientations: int = 1
    pool: str = "none"
    pool_group: int = 4
    convention: str = "scatter"

    def c(self) -> _Desc:
        return _Desc(self.n, self.c_in, self.h, self.w, self.c_out, self.k, GROUPS[self.group],
                     self.orientations, POOLS[self.pool], self.pool_group,
                     CONVENTIONS[self.convention])

    @property
    def num_bases(self) -> int:
        return {"single": 1, "p4": 1, "p4m": 2, "steer": self.orientations // 4}[self.group]

    @property
    def out_orientations(self) -> int:
        R = self.orientations
        return {"none": R, "avg": 1, "max": 1, "subgroup": R // self.pool_group}[self.pool]

    @property
    def has_argmax(self) -> bool:
        return self.pool in ("max", "subgroup")


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle library missing: {ORACLE_SO} (run make -C oracle)")
        _lib = C.CDLL(ORACLE_SO)
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference build missing: {REF_SO}")
        _ref = C.CDLL(REF_SO)
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _sfx(dtype) -> str:
    return "f" if np.dtype(dtype) == np.float32 else "d"


# ---------------------------------------------------------------- oracle (C restatement)

def validate(d: Desc) -> str | None:
    buf = C.create_string_buffer(256)
    dd = d.c()
    rc = lib().rco_validate(C.byref(dd), buf, C.c_size_t(256))
    return None if rc == 0 else buf.value.decode()


def slice_tap_map(k: int, r: int, convention: str = "scatter") -> np.ndarray:
    m = np.zeros(k * k, np.int32)
    lib().rco_slice_tap_map(k, r, CONVENTIONS[convention], _p(m))
    return m.reshape(k, k)


def clipped_writes(h, w, kh, kw) -> int:
    f = lib().rco_clipped_writes
    f.restype = C.c_ulonglong
    return int(f(h, w, kh, kw))


def rot90_plane(a: np.ndarray, q: int) -> np.ndarray:
    a = np.ascontiguousarray(a)
    out = np.empty(a.size, a.dtype)
    r, c = C.c_int(), C.c_int()
    getattr(lib(), "rco_rot90_plane_" + _sfx(a.dtype))(_p(a), a.shape[0], a.shape[1], q, _p(out),
                                                      C.byref(r), C.byref(c))
    return out.reshape(r.value, c.value)


def mirror_plane(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    out = np.empty_like(a)
    getattr(lib(), "rco_mirror_plane_" + _sfx(a.dtype))(_p(a), a.shape[0], a.shape[1], _p(out))
    return out


def transform_kernel(w: np.ndarray, r: int, mirror: bool = False) -> np.ndarray:
    w = np.ascontiguousarray(w)
    out = np.empty_like(w)
    getattr(lib(), "rco_transform_kernel_" + _sfx(w.dtype))(
        _p(w), w.shape[0], w.shape[1], w.shape[2], r, int(mirror), _p(out))
    return out


def steer(fx: np.ndarray, fy: np.ndarray, theta: float) -> np.ndarray:
    fx, fy = np.ascontiguousarray(fx), np.ascontiguousarray(fy)
    out = np.empty_like(fx)
    getattr(lib(), "rco_steer_" + _sfx(fx.dtype))(_p(fx), _p(fy), C.c_size_t(fx.size),
                                                 C.c_double(theta), _p(out))
    return out


def build_bases(d: Desc, w0: np.ndarray, w1: np.ndarray | None = None) -> np.ndarray:
    w0 = np.ascontiguousarray(w0)
    w1 = np.ascontiguousarray(w1) if w1 is not None else w0
    out = np.empty((d.num_bases,) + w0.shape, w0.dtype)
    dd = d.c()
    getattr(lib(), "rco_build_bases_" + _sfx(w0.dtype))(C.byref(dd), _p(w0), _p(w1), _p(out))
    return out


def build_orientation_bank(d: Desc, w0: np.ndarray, w1: np.ndarray | None = None) -> np.ndarray:
    w0 = np.ascontiguousarray(w0)
    w1 = np.ascontiguousarray(w1) if w1 is not None else w0
    out = np.empty((d.orientations,) + w0.shape, w0.dtype)
    dd = d.c()
    getattr(lib(), "rco_build_orientation_bank_" + _sfx(w0.dtype))(C.byref(dd), _p(w0), _p(w1),
                                                                  _p(out))
    return out


def scatter_conv_single(x: np.ndarray, k: np.ndarray):
    x, k = np.ascontiguousarray(x), np.ascontiguousarray(k)
    y = np.empty_like(x)
    m, a = C.c_ulonglong(0), C.c_ulonglong(0)
    getattr(lib(), "rco_scatter_conv_single_" + _sfx(x.dtype))(
        _p(x), x.shape[0], x.shape[1], _p(k), k.shape[0], k.shape[1], _p(y), C.byref(m),
        C.byref(a))
    return y, m.value, a.value


def _conv(name, x, w):
    x, w = np.ascontiguousarray(x), np.ascontiguousarray(w)
    cin, h, ww = x.shape
    cout, _, kh, kw = w.shape
    y = np.empty((cout, h, ww), x.dtype)
    getattr(lib(), name + "_" + _sfx(x.dtype))(_p(x), cin, h, ww, _p(w), cout, kh, kw, _p(y))
    return y


def scatter_conv_multi(x, w):
    return _conv("rco_scatter_conv_multi", x, w)


def scatter_conv_raw_multi(x, w):
    return _conv("rco_scatter_conv_raw_multi", x, w)


def conv_gather_same(x, w):
    return _conv("rco_conv_gather_same", x, w)


def group_conv_scatter_reuse(d: Desc, x: np.ndarray, bases: np.ndarray) -> np.ndarray:
    x, bases = np.ascontiguousarray(x), np.ascontiguousarray(bases)
    f = np.empty((d.c_out, d.orientations, d.h, d.w), x.dtype)
    dd = d.c()
    getattr(lib(), "rco_group_conv_scatter_reuse_" + _sfx(x.dtype))(C.byref(dd), _p(x), _p(bases),
                                                                   _p(f))
    return f


def orientation_pool_avg(f: np.ndarray) -> np.ndarray:
    f = np.ascontiguousarray(f)
    co, r, h, w = f.shape
    y = np.empty((co, h, w), f.dtype)
    getattr(lib(), "rco_orientation_pool_avg_" + _sfx(f.dtype))(_p(f), co, r, h, w, _p(y))
    return y


def orientation_pool_max(f: np.ndarray):
    f = np.ascontiguousarray(f)
    co, r, h, w = f.shape
    y = np.empty((co, h, w), f.dtype)
    a = np.empty((co, h, w), np.uint8)
    getattr(lib(), "rco_orientation_pool_max_" + _sfx(f.dtype))(_p(f), co, r, h, w, _p(y), _p(a))
    return y, a


def subgroup_pool_max(f: np.ndarray, g: int = 4):
    f = np.ascontiguousarray(f)
    co, r, h, w = f.shape
    y = np.empty((co, r // g, h, w), f.dtype)
    a = np.empty((co, r // g, h, w), np.uint8)
    getattr(lib(), "rco_subgroup_pool_max_" + _sfx(f.dtype))(_p(f), co, r, h, w, g, _p(y), _p(a))
    return y, a


def ri_forward(d: Desc, x: np.ndarray, w0: np.ndarray, w1: np.ndarray | None = None,
               bias: np.ndarray | None = None, nthreads: int = 1, images: tuple | None = None):
    """Full layer over the batch (or images=(begin, end)): returns (y, argmax|None).

    x: (N, Cin, H, W); y: (N, Cout, R', H, W) (R' squeezed away for avg/max pools).
    """
    x = np.ascontiguousarray(x)
    w0 = np.ascontiguousarray(w0)
    w1 = np.ascontiguousarray(w1) if w1 is not None else w0
    ro = d.out_orientations
    y = np.zeros((d.n, d.c_out, ro, d.h, d.w), x.dtype)
    a = np.zeros((d.n, d.c_out, ro, d.h, d.w), np.uint8) if d.has_argmax else None
    b = np.ascontiguousarray(bias, x.dtype) if bias is not None else None
    b0, b1 = images if images is not None else (0, d.n)
    dd = d.c()
    rc = getattr(lib(), "rco_ri_forward_" + _sfx(x.dtype))(
        C.byref(dd), _p(x), _p(w0), _p(w1), _p(b) if b is not None else None, _p(y),
        _p(a) if a is not None else None, nthreads, b0, b1)
    if rc != 0:
        raise ValueError(validate(d))
    if d.pool in ("avg", "max"):
        y = y[:, :, 0]
        a = a[:, :, 0] if a is not None else None
    return y, a


# ---------------------------------------------------------------- reference (_ref) bindings

def ref_scatter_conv_multi(x, w):
    x, w = np.ascontiguousarray(x), np.ascontiguousarray(w)
    cin, h, ww = x.shape
    cout, _, kh, kw = w.shape
    y = np.empty((cout, h, ww), x.dtype)
    m = C.c_ulonglong(0)
    getattr(ref(), "ref_scatter_conv_multi_" + _sfx(x.dtype))(_p(x), cin, h, ww, _p(w), cout, kh,
                                                             kw, _p(y), C.byref(m))
    return y, m.value


def ref_scatter_conv_raw_multi(x, w):
    x, w = np.ascontiguousarray(x), np.ascontiguousarray(w)
    cin, h, ww = x.shape
    cout, _, kh, kw = w.shape
    y = np.empty((cout, h, ww), x.dtype)
    getattr(ref(), "ref_scatter_conv_raw_multi_" + _sfx(x.dtype))(_p(x), cin, h, ww, _p(w), cout,
                                                                 kh, kw, _p(y))
    return y


def ref_conv_gather_same(x, w):
    x, w = np.ascontiguousarray(x), np.ascontiguousarray(w)
    cin, h, ww = x.shape
    cout, _, kh, kw = w.shape
    y = np.empty((cout, h, ww), x.dtype)
    getattr(ref(), "ref_conv_gather_same_" + _sfx(x.dtype))(_p(x), cin, h, ww, _p(w), cout, kh, kw,
                                                           _p(y))
    return y


def ref_tiled_scatter_conv(x, w, tile=(32, 32), halo=None, workers=1, strategy=0):
    """Returns (y, mults, adds, aux_peak); raises ValueError with the reference message."""
    x, w = np.ascontiguousarray(x), np.ascontiguousarray(w)
    cin, h, ww = x.shape
    cout, cin_w, kh, kw = w.shape
    halo = kh // 2 if halo is None else halo
    y = np.empty((cout, h, ww), x.dtype)
    m, a, aux = C.c_ulonglong(0), C.c_ulonglong(0), C.c_ulonglong(0)
    err = C.create_string_buffer(256)
    rc = getattr(ref(), "ref_tiled_scatter_conv_" + _sfx(x.dtype))(
        _p(x), cin, h, ww, _p(w), cout, cin_w, kh, kw, tile[0], tile[1], halo, workers, strategy, _p(y),
        C.byref(m), C.byref(a), C.byref(aux), err, C.c_size_t(256))
    if rc != 0:
        raise ValueError(err.value.decode())
    return y, m.value, a.value, aux.value


def ref_ri_slices(d: Desc, x: np.ndarray, w0: np.ndarray, bases: np.ndarray | None = None):
    """Unpooled (Cout, R, H, W) from reference primitives (R x tiled_scatter_conv)."""
    x = np.ascontiguousarray(x)
    src = np.ascontiguousarray(bases if d.group == "steer" else w0)
    f = np.empty((d.c_out, d.orientations, d.h, d.w), x.dtype)
    getattr(ref(), "ref_ri_slices_" + _sfx(x.dtype))(
        GROUPS[d.group], d.orientations, CONVENTIONS[d.convention], _p(x), d.c_in, d.h, d.w,
        _p(src), d.c_out, d.k, _p(f))
    return f


def ref_ri_batch(d: Desc, x: np.ndarray, w0: np.ndarray, w1: np.ndarray | None = None,
                 bias: np.ndarray | None = None, nthreads: int = 1, images: tuple | None = None):
    """The RI layer on the reference's own code path: R x tiled_scatter_conv per image
    (ref_ri_slices) + the SPEC pooling and bias.  Same shapes as ri_forward (float32)."""
    x = np.ascontiguousarray(x, np.float32)
    w0 = np.ascontiguousarray(w0, np.float32)
    src = np.ascontiguousarray(build_bases(d, w0, w1 if w1 is not None else w0), np.float32) \
        if d.group == "steer" else w0
    ro = d.out_orientations
    y = np.zeros((d.n, d.c_out, ro, d.h, d.w), np.float32)
    a = np.zeros((d.n, d.c_out, ro, d.h, d.w), np.uint8) if d.has_argmax else None
    b = np.ascontiguousarray(bias, np.float32) if bias is not None else None
    b0, b1 = images if images is not None else (0, d.n)
    ref().ref_ri_batch_f(GROUPS[d.group], d.orientations, CONVENTIONS[d.convention], POOLS[d.pool],
                         d.pool_group, _p(x), d.n, d.c_in, d.h, d.w, _p(src), d.c_out, d.k,
                         _p(b) if b is not None else None, _p(y), _p(a) if a is not None else None,
                         nthreads, b0, b1)
    if d.pool in ("avg", "max"):
        y = y[:, :, 0]
        a = a[:, :, 0] if a is not None else None
    return y, a


def ref_tiled_batch(x: np.ndarray, w: np.ndarray, nthreads: int, images: tuple):
    x, w = np.ascontiguousarray(x, np.float32), np.ascontiguousarray(w, np.float32)
    n, c, h, ww = x.shape
    cout, _, k, _ = w.shape
    y = np.zeros((n, cout, h, ww), np.float32)
    ref().ref_tiled_batch_f(_p(x), n, c, h, ww, _p(w), cout, k, _p(y), nthreads, images[0],
                            images[1])
    return y
