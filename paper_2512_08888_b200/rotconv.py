"""Python mirror of the reference's rotconv API over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference C++ headers
(/root/reference/proj/include/rotconv/*.hpp) and the SPEC-defined RI ops that have no
shipped code (SPEC.md group_conv / steerable modules):

    reference (C++, CPU)                               here (torch CUDA tensors)
    tiled_scatter_conv        scatter_conv.hpp:330-368 tiled_scatter_conv
    scatter_conv_multi        scatter_conv.hpp:189-193 scatter_conv_multi
    scatter_conv_raw_multi    scatter_conv.hpp:151-187 scatter_conv_raw_multi
    scatter_conv_single       scatter_conv.hpp:143-149 scatter_conv_single
    transform_kernel          SPEC:256-264             transform_kernel
    group_conv_scatter_reuse  SPEC:274-282             group_conv_scatter_reuse
    orientation_pool_avg/max  SPEC:283-300             orientation_pool_avg / _max
    subgroup_pool_max         SPEC:301-309             subgroup_pool_max
    steer                     SPEC:439-447             steer
    build_orientation_bank    SPEC:448-456             build_orientation_bank
    (north star) fused layer                           ri_conv / RIConv

Tensors are the reference containers' layouts: Tensor3 (C,H,W), FilterBank
(Cout,Cin,K,K), OrientedFeature (Cout,R,H,W); a leading batch dim N is accepted
everywhere.  Preconditions raise ValueError with the reference's message strings
(std::invalid_argument); CUDA failures raise RotconvError.  Every op runs the sm_100a
kernels in librotconv_b200.so -- inputs must be float32 CUDA tensors.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum

import torch

from . import _lib
from ._lib import check, lib, rc_desc


# ----------------------------------------------------------------------------- types
@dataclass
class MultCounter:
    """scatter_conv.hpp:28-41 -- analytic op counts, accumulated (add, never reset)."""
    scalar_multiplications: int = 0
    scalar_additions: int = 0

    def add(self, mults: int, adds: int) -> None:
        self.scalar_multiplications += int(mults)
        self.scalar_additions += int(adds)

    def reset(self) -> None:
        self.scalar_multiplications = 0
        self.scalar_additions = 0


@dataclass
class AuxMemCounter:
    """scatter_conv.hpp:43-57 -- high-water mark of auxiliary (device workspace) bytes."""
    current_bytes: int = 0
    peak_bytes: int = 0

    def acquire(self, n: int) -> None:
        self.current_bytes += n
        self.peak_bytes = max(self.peak_bytes, self.current_bytes)

    def release(self, n: int) -> None:
        self.current_bytes = 0 if n > self.current_bytes else self.current_bytes - n

    def reset(self) -> None:
        self.current_bytes = self.peak_bytes = 0


@dataclass
class TileConfig:
    """scatter_conv.hpp:59-65 (tile/halo are validated; the GPU result is tile-invariant)."""
    tile_h: int = 32
    tile_w: int = 32
    halo: int = 1


class ScatterStrategy(Enum):
    tile_private = 0
    phase_parallel = 1


@dataclass(frozen=True)
class GroupSpec:
    """kind p4 (size 4) or p4m (size 8)."""
    kind: str = "p4"

    @property
    def size(self) -> int:
        return {"p4": 4, "p4m": 8}[self.kind]


@dataclass
class SteerableBasis:
    """paired base banks f_x, f_y of identical shape (Cout,Cin,K,K)."""
    f_x: torch.Tensor
    f_y: torch.Tensor


@dataclass
class Desc:
    """Python view of rc_desc (include/rotconv_c.h)."""
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
    precision: str = "auto"
    activation: str = "none"

    def c(self) -> rc_desc:
        return rc_desc(self.n, self.c_in, self.h, self.w, self.c_out, self.k,
                       _lib.GROUPS[self.group], self.orientations, _lib.POOLS[self.pool],
                       self.pool_group, _lib.CONVENTIONS[self.convention],
                       _lib.PRECISIONS[self.precision], _lib.ACTIVATIONS[self.activation])

    def validate(self) -> None:
        d = self.c()
        check(lib().rc_validate(C.byref(d)))

    @property
    def num_bases(self) -> int:
        return {"single": 1, "p4": 1, "p4m": 2, "steer": self.orientations // 4}[self.group]

    @property
    def out_orientations(self) -> int:
        d = self.c()
        return lib().rc_out_orientations(C.byref(d))

    @property
    def has_argmax(self) -> bool:
        return self.pool in ("max", "subgroup")

    def bank_bytes(self) -> int:
        d = self.c()
        return int(lib().rc_bank_bytes(C.byref(d)))

    def workspace_bytes(self) -> int:
        d = self.c()
        return int(lib().rc_workspace_size(C.byref(d)))

    def kernel_name(self) -> str | None:
        d = self.c()
        r = lib().rc_kernel_name(C.byref(d))
        return r.decode() if r else None

    def analytic_counts(self) -> tuple[int, int]:
        d = self.c()
        m, a = C.c_ulonglong(0), C.c_ulonglong(0)
        check(lib().rc_analytic_counts(C.byref(d), C.byref(m), C.byref(a)))
        return m.value, a.value

    # FLOP figures used by bench.py / DESIGN.md
    def alg_flops(self) -> int:
        return 2 * self.n * self.h * self.w * self.k * self.k * self.c_in * self.c_out * self.num_bases

    def eff_flops(self) -> int:
        return 2 * self.n * self.h * self.w * self.k * self.k * self.c_in * self.c_out * self.orientations


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device: torch.device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check_cuda_f32(name: str, t: torch.Tensor) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor (the product path runs only on the GPU)")
    if t.dtype != torch.float32:
        raise TypeError(f"{name}: expected float32 (the reference's benchmark mode)")
    return t.contiguous()


def clipped_writes(h: int, w: int, kh: int, kw: int) -> int:
    """scatter_conv.hpp:94-110."""
    return int(lib().rc_clipped_writes(h, w, kh, kw))


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    b, e = C.c_int(), C.c_int()
    check(lib().rc_shard_range(n, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


# ----------------------------------------------------------------------- bank + layer
def bank_precompute(desc: Desc, w0: torch.Tensor, w1: torch.Tensor | None = None) -> torch.Tensor:
    """Rotated-filter-bank precompute: opaque device bank (uint8)."""
    desc.validate()
    w0 = _check_cuda_f32("w0", w0)
    if desc.group == "steer":
        if w1 is None:
            raise ValueError("SteerableBasis: f_x and f_y are required")
        w1 = _check_cuda_f32("w1", w1)
        if w1.shape != w0.shape:
            raise ValueError("SteerableBasis: f_x and f_y shapes must be equal")
    if tuple(w0.shape) != (desc.c_out, desc.c_in, desc.k, desc.k):
        raise ValueError("ri_conv: weight shape must be (Cout, Cin, K, K)")
    bank = torch.empty(desc.bank_bytes(), dtype=torch.uint8, device=w0.device)
    d = desc.c()
    check(lib().rc_bank_precompute(C.byref(d), _ptr(w0), _ptr(w1), _ptr(bank), _stream(w0.device)))
    return bank


def bank_bases(desc: Desc, bank: torch.Tensor) -> torch.Tensor:
    """View of the bank's base kernels K_b: (B, Cout, Cin, K, K) float32."""
    nb = desc.num_bases * desc.c_out * desc.c_in * desc.k * desc.k
    return bank[: nb * 4].view(torch.float32).view(desc.num_bases, desc.c_out, desc.c_in, desc.k, desc.k)


def ri_conv_forward(desc: Desc, x: torch.Tensor, bank: torch.Tensor,
                    bias: torch.Tensor | None = None, out: torch.Tensor | None = None,
                    argmax: torch.Tensor | None = None):
    """The fused layer: reuse scatter + orientation reduction + bias, one launch.

    x: (N, Cin, H, W) float32 CUDA.  Returns (y, argmax|None) with y of shape
    (N, Cout, R', H, W) (R' = out orientations).
    """
    desc.validate()
    x = _check_cuda_f32("x", x)
    if tuple(x.shape) != (desc.n, desc.c_in, desc.h, desc.w):
        raise ValueError("ri_conv: input shape must be (N, Cin, H, W) of the descriptor")
    if bias is not None:
        bias = _check_cuda_f32("bias", bias)
        if bias.numel() != desc.c_out:
            raise ValueError("ri_conv: bias must have Cout elements")
    ro = desc.out_orientations
    shape = (desc.n, desc.c_out, ro, desc.h, desc.w)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=x.device)
    if desc.has_argmax and argmax is None:
        argmax = torch.empty(shape, dtype=torch.uint8, device=x.device)
    ws_bytes = desc.workspace_bytes()
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)
    d = desc.c()
    check(lib().rc_ri_conv_forward(C.byref(d), _ptr(x), _ptr(bank), _ptr(bias), _ptr(out),
                                   _ptr(argmax) if desc.has_argmax else None, _ptr(ws),
                                   C.c_size_t(ws_bytes), _stream(x.device)))
    return out, (argmax if desc.has_argmax else None)


def ri_conv(x: torch.Tensor, w0: torch.Tensor, w1: torch.Tensor | None = None, *,
            group: str = "steer", orientations: int = 8, pool: str = "subgroup",
            pool_group: int = 4, bias: torch.Tensor | None = None, convention: str = "scatter",
            precision: str = "auto", counter: MultCounter | None = None):
    """Whole RI layer (bank precompute + fused forward) on a batch (N,Cin,H,W)."""
    squeeze = x.dim() == 3
    xb = x.unsqueeze(0) if squeeze else x
    n, cin, h, w = xb.shape
    desc = Desc(n, cin, h, w, w0.shape[0], w0.shape[2], group, orientations, pool, pool_group,
                convention, precision)
    if w0.shape[1] != cin:
        raise ValueError("ri_conv: channel mismatch")
    bank = bank_precompute(desc, w0, w1)
    y, a = ri_conv_forward(desc, xb, bank, bias)
    if counter is not None:
        counter.add(*desc.analytic_counts())
    if pool in ("avg", "max"):
        y = y[:, :, 0]
        a = a[:, :, 0] if a is not None else None
    if squeeze:
        y = y[0]
        a = a[0] if a is not None else None
    return y, a


class RIConv:
    """Stateful layer: weights + precomputed bank, reused across forwards."""

    def __init__(self, w0, w1=None, *, group="steer", orientations=8, pool="subgroup",
                 pool_group=4, bias=None, convention="scatter", precision="auto"):
        self.w0, self.w1, self.bias = w0, w1, bias
        self.kw = dict(group=group, orientations=orientations, pool=pool, pool_group=pool_group,
                       convention=convention, precision=precision)
        self._bank = None
        self._bank_key = None

    def desc(self, n, h, w) -> Desc:
        return Desc(n, self.w0.shape[1], h, w, self.w0.shape[0], self.w0.shape[2], **self.kw)

    def _weights_key(self):
        # the bank depends only on the weight values (not on N, H or W): rebuild it when a
        # weight tensor is replaced or updated in place (an optimizer step bumps _version)
        return tuple((t.data_ptr(), t._version) if t is not None else None for t in (self.w0, self.w1))

    def refresh_bank(self) -> None:
        """Drop the cached bank; the next call rebuilds it from the current weights."""
        self._bank = None
        self._bank_key = None

    def __call__(self, x: torch.Tensor):
        n, _, h, w = x.shape
        desc = self.desc(n, h, w)
        key = self._weights_key()
        if self._bank is None or self._bank_key != key:
            self._bank = bank_precompute(desc, self.w0, self.w1)
            self._bank_key = key
        return ri_conv_forward(desc, x, self._bank, self.bias)


# ------------------------------------------------------------- reference-named operations
# Precision of the reference-named drop-ins, which have no precision argument in the
# reference signatures: "auto" (the FP32-tolerance tensor-core kernels where the shape has
# one) unless the caller passes precision= explicitly (e.g. "fp32" for the CUDA-core FFMA
# path, bit-identical to the reference on exactly representable inputs).
DEFAULT_PRECISION = "auto"


def _single_desc(x: torch.Tensor, w: torch.Tensor, convention: str,
                 precision: str | None = None) -> tuple[Desc, torch.Tensor, bool]:
    squeeze = x.dim() == 3
    xb = x.unsqueeze(0) if squeeze else x
    n, cin, h, ww = xb.shape
    return (Desc(n, cin, h, ww, w.shape[0], w.shape[2], "single", 1, "none", 1, convention,
                 precision or DEFAULT_PRECISION), xb, squeeze)


def _run_single(x, w, convention, name, precision=None):
    if w.shape[1] != x.shape[-3]:
        raise ValueError(f"{name}: channel mismatch")
    if w.shape[2] != w.shape[3]:
        raise ValueError(f"{name}: kernel must be square")
    desc, xb, squeeze = _single_desc(x, w, convention, precision)
    bank = bank_precompute(desc, w)
    y, _ = ri_conv_forward(desc, xb, bank)
    y = y[:, :, 0]
    return y[0] if squeeze else y


def scatter_conv_multi(x: torch.Tensor, w: torch.Tensor, counter: MultCounter | None = None, *,
                       precision: str | None = None):
    """scatter_conv.hpp:189-193: equals conv_gather_same(x, reverse_bank(w))."""
    y = _run_single(x, w, "scatter", "scatter_conv_multi", precision)
    if counter is not None:
        n = 1 if x.dim() == 3 else x.shape[0]
        h, ww = x.shape[-2:]
        counter.add(n * h * ww * w.shape[2] * w.shape[3] * w.shape[1] * w.shape[0],
                    n * clipped_writes(h, ww, w.shape[2], w.shape[3]) * w.shape[0])
    return y


def scatter_conv_raw_multi(x: torch.Tensor, w: torch.Tensor, counter: MultCounter | None = None, *,
                           precision: str | None = None):
    """scatter_conv.hpp:151-187: raw scatter indices, equals conv_gather_same(x, w)."""
    y = _run_single(x, w, "raw", "scatter_conv_multi", precision)
    if counter is not None:
        n = 1 if x.dim() == 3 else x.shape[0]
        h, ww = x.shape[-2:]
        counter.add(n * h * ww * w.shape[2] * w.shape[3] * w.shape[1] * w.shape[0],
                    n * clipped_writes(h, ww, w.shape[2], w.shape[3]) * w.shape[0])
    return y


def scatter_conv_single(x: torch.Tensor, k: torch.Tensor, counter: MultCounter | None = None, *,
                        precision: str | None = None):
    """scatter_conv.hpp:143-149: single plane (H,W) with an arbitrary (Kh,Kw) kernel."""
    if k.shape[0] != k.shape[1]:
        # the reference supports rectangular single-plane kernels; the GPU kernels
        # are square-only, so refuse rather than silently differ
        raise ValueError("scatter_conv_single: kernel must be square on the GPU path")
    y = _run_single(x.reshape(1, 1, *x.shape), k.reshape(1, 1, *k.shape), "scatter",
                    "scatter_conv_single", precision)[0, 0]
    if counter is not None:
        counter.add(x.shape[0] * x.shape[1] * k.shape[0] * k.shape[1],
                    clipped_writes(x.shape[0], x.shape[1], k.shape[0], k.shape[1]))
    return y


def tiled_scatter_conv(x: torch.Tensor, w: torch.Tensor, cfg: TileConfig, workers: int,
                       counter: MultCounter | None = None, aux: AuxMemCounter | None = None,
                       strategy: ScatterStrategy = ScatterStrategy.tile_private, *,
                       precision: str | None = None):
    """scatter_conv.hpp:330-368 -- the shipped drop-in entry point (R = 1).

    AuxMemCounter follows the reference's accounting (:351-360): tile_private acquires and
    releases tile_h * tile_w * sizeof(float) * workers bytes; phase_parallel none."""
    cin = x.shape[-3]
    if cin != w.shape[1]:
        raise ValueError("tiled_scatter_conv: channel mismatch")
    if w.shape[2] != w.shape[3]:
        raise ValueError("tiled_scatter_conv: kernel must be square")
    if cfg.tile_h < 1 or cfg.tile_w < 1:
        raise ValueError("tiled_scatter_conv: tile dims must be >= 1")
    if cfg.halo != w.shape[2] // 2:
        raise ValueError("tiled_scatter_conv: invalid halo")
    if workers < 1:
        raise ValueError("tiled_scatter_conv: workers must be >= 1")
    desc, xb, squeeze = _single_desc(x, w, "scatter", precision)
    aux_bytes = cfg.tile_h * cfg.tile_w * 4 * workers
    if aux is not None and strategy == ScatterStrategy.tile_private:
        aux.acquire(aux_bytes)
    bank = bank_precompute(desc, w)
    y, _ = ri_conv_forward(desc, xb, bank)
    if aux is not None and strategy == ScatterStrategy.tile_private:
        aux.release(aux_bytes)
    if counter is not None:
        counter.add(*desc.analytic_counts())
    y = y[:, :, 0]
    return y[0] if squeeze else y


def transform_kernel(w: torch.Tensor, r: int, mirror: bool = False) -> torch.Tensor:
    """SPEC:256-264 via the bank kernel: mirror (p4m) then r CCW quarter turns."""
    if w.shape[-1] != w.shape[-2] and r % 2 == 1:
        raise ValueError("transform_kernel: rotation needs a square kernel")
    desc = Desc(1, w.shape[1], 1, 1, w.shape[0], w.shape[2], "p4m" if mirror else "p4",
                8 if mirror else 4)
    if w.shape[2] % 2 == 0:  # even kernels: the p4/p4m bank requires odd K; rotate on the host side
        out = w
        if mirror:
            out = torch.flip(out, dims=[-1])
        return torch.rot90(out, k=r % 4, dims=(-2, -1)).contiguous()
    kernels = build_orientation_bank_from(desc, w)
    return kernels[(4 if mirror else 0) + (r % 4)]


def build_orientation_bank_from(desc: Desc, w0: torch.Tensor, w1: torch.Tensor | None = None) -> torch.Tensor:
    bank = bank_precompute(desc, w0, w1)
    out = torch.empty((desc.orientations,) + tuple(w0.shape), dtype=torch.float32, device=w0.device)
    d = desc.c()
    check(lib().rc_orientation_bank(C.byref(d), _ptr(bank), _ptr(out), _stream(w0.device)))
    return out


def steer(basis: SteerableBasis, theta: float) -> torch.Tensor:
    """sin(theta) f_x + cos(theta) f_y (coefficients rounded from double)."""
    fx = _check_cuda_f32("f_x", basis.f_x)
    fy = _check_cuda_f32("f_y", basis.f_y)
    s = torch.tensor(float(math.sin(theta)), dtype=torch.float32, device=fx.device)
    c = torch.tensor(float(math.cos(theta)), dtype=torch.float32, device=fx.device)
    return s * fx + c * fy


def build_orientation_bank(basis: SteerableBasis, n: int):
    """(kernels[R], tags[(base_angle, quadrant r)]) orbit-major."""
    if n < 4 or n % 4 != 0:
        raise ValueError("build_orientation_bank: N must be a multiple of 4")
    fx = basis.f_x
    desc = Desc(1, fx.shape[1], 1, 1, fx.shape[0], fx.shape[2], "steer", n)
    kernels = build_orientation_bank_from(desc, basis.f_x, basis.f_y)
    tags = [(2 * math.pi * b / n, r) for b in range(n // 4) for r in range(4)]
    return kernels, tags


def group_conv_scatter_reuse(x: torch.Tensor, w: torch.Tensor, g: GroupSpec,
                             counter: MultCounter | None = None, *,
                             precision: str | None = None) -> torch.Tensor:
    """SPEC:274-282 -> OrientedFeature (Cout, |G|, H, W) (batched: leading N)."""
    y, _ = ri_conv(x, w, None, group=g.kind, orientations=g.size, pool="none", counter=counter,
                   precision=precision or DEFAULT_PRECISION)
    return y


def _pool(f: torch.Tensor, pool: str, g: int):
    f = _check_cuda_f32("F", f)
    squeeze = f.dim() == 4
    fb = f.unsqueeze(0) if squeeze else f
    n, co, r, h, w = fb.shape
    gf = r if pool in ("avg", "max") else g
    if pool == "subgroup" and (g < 1 or r % g != 0):
        raise ValueError("subgroup_pool_max: R not divisible by group_size")
    ro = r // gf
    y = torch.empty((n, co, ro, h, w), dtype=torch.float32, device=f.device)
    a = torch.empty((n, co, ro, h, w), dtype=torch.uint8, device=f.device) if pool != "avg" else None
    check(lib().rc_orientation_pool(n, co, r, h, w, _lib.POOLS[pool], g, _ptr(fb), None, _ptr(y),
                                    _ptr(a), _stream(f.device)))
    if pool in ("avg", "max"):
        y = y[:, :, 0]
        a = a[:, :, 0] if a is not None else None
    if squeeze:
        y = y[0]
        a = a[0] if a is not None else None
    return y, a


def orientation_pool_avg(f: torch.Tensor) -> torch.Tensor:
    """SPEC:283-291 Eq. (9)."""
    return _pool(f, "avg", 1)[0]


def orientation_pool_max(f: torch.Tensor):
    """SPEC:292-300 Eq. (10): (values, argmax) with ties -> smallest r."""
    return _pool(f, "max", 1)


def subgroup_pool_max(f: torch.Tensor, group_size: int = 4):
    """blockwise max over contiguous blocks, block-local argmax."""
    return _pool(f, "subgroup", group_size)


# ------------------------------------------------- steerable regularisers
# Training-side scalars over the B filter pairs of a basis: tiny reductions
# over the weights, computed with torch ops wherever the basis lives.  Not on the forward
# hot path.
def gaussian_derivative_basis(k: int, sigma: float, out_channels: int = 1, in_channels: int = 1,
                              device="cpu", dtype=torch.float64) -> SteerableBasis:
    """f_x ~ -x exp(-(x^2+y^2)/2s^2), f_y ~ -y exp(..), unit L2, centred grid."""
    if k < 1 or k % 2 == 0:
        raise ValueError("gaussian_derivative_basis: K must be odd")
    if sigma <= 0:
        raise ValueError("gaussian_derivative_basis: sigma must be positive")
    c = k // 2
    ax = torch.arange(k, dtype=torch.float64) - c
    yy, xx = torch.meshgrid(ax, ax, indexing="ij")
    g = torch.exp(-(xx * xx + yy * yy) / (2 * sigma * sigma))
    fx, fy = -xx * g, -yy * g
    fx, fy = fx / fx.norm(), fy / fy.norm()
    shape = (out_channels, in_channels, k, k)
    return SteerableBasis(fx.expand(shape).to(device=device, dtype=dtype).contiguous(),
                          fy.expand(shape).to(device=device, dtype=dtype).contiguous())


def loss_mag(basis: SteerableBasis) -> torch.Tensor:
    """SPEC:457-466 Eq. (19): mean over filters b of (||w_x_b|| - ||w_y_b||)^2."""
    nx = basis.f_x.reshape(basis.f_x.shape[0], -1).double().norm(dim=1)
    ny = basis.f_y.reshape(basis.f_y.shape[0], -1).double().norm(dim=1)
    return ((nx - ny) ** 2).mean()


def loss_orth(basis: SteerableBasis, eps: float = 1e-8) -> torch.Tensor:
    """SPEC:467-474 Eq. (20): mean over b of (<w_x, w_y> / (||w_x|| ||w_y|| + eps))^2."""
    if eps <= 0:
        raise ValueError("loss_orth: eps must be positive")
    x = basis.f_x.reshape(basis.f_x.shape[0], -1).double()
    y = basis.f_y.reshape(basis.f_y.shape[0], -1).double()
    c = (x * y).sum(dim=1) / (x.norm(dim=1) * y.norm(dim=1) + eps)
    return (c ** 2).mean()


def total_loss(ce, basis: SteerableBasis, lambda_mag: float, lambda_orth: float, eps: float = 1e-8):
    """SPEC:475-483 Eq. (18): ce + lambda_mag * L_mag + lambda_orth * L_orth."""
    if lambda_mag < 0 or lambda_orth < 0:
        raise ValueError("total_loss: lambdas must be >= 0")
    return ce + lambda_mag * loss_mag(basis) + lambda_orth * loss_orth(basis, eps)


# ------------------------------------------------------------ backward
def ri_conv_backward(desc: Desc, x: torch.Tensor, bank: torch.Tensor, gy: torch.Tensor,
                     y: torch.Tensor | None = None, argmax: torch.Tensor | None = None,
                     need_input: bool = True, need_weight: bool = True, need_bias: bool = True):
    """Gradients of ri_conv_forward for the upstream gradient gy (N, Cout, R', H, W).

    Returns (dx | None, dw0 | None, dw1 | None, dbias | None): dw0 = dW (single, p4, p4m) or
    d f_x (steer), dw1 = d f_y (steer).  y (the forward output) is needed for ReLU layers,
    argmax for max / subgroup pooling.  gy is not modified (a masked copy is used).
    """
    desc.validate()
    x = _check_cuda_f32("x", x)
    gy = _check_cuda_f32("gy", gy).clone()  # the C-ABI masks it in place for ReLU
    dev = x.device
    d = desc.c()
    L = lib()
    scratch = torch.empty(int(L.rc_backward_scratch_bytes(C.byref(d))) // 4 or 1, device=dev)
    wsb = int(L.rc_backward_workspace_size(C.byref(d)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    dx = torch.empty_like(x) if need_input else None
    wshape = (desc.c_out, desc.c_in, desc.k, desc.k)
    dw0 = torch.empty(wshape, device=dev) if need_weight else None
    dw1 = torch.empty(wshape, device=dev) if (need_weight and desc.group == "steer") else None
    db = torch.empty(desc.c_out, device=dev) if need_bias else None
    check(L.rc_ri_conv_backward(C.byref(d), _ptr(x), _ptr(bank), _ptr(y), _ptr(gy), _ptr(argmax), _ptr(dx),
                                _ptr(dw0), _ptr(dw1), _ptr(db), _ptr(scratch), _ptr(ws), C.c_size_t(wsb),
                                _stream(dev)))
    return dx, dw0, dw1, db


class RIConvFunction(torch.autograd.Function):
    """autograd bridge: y = fused RI layer(x; w0, w1, bias), backward through the C-ABI.

    ``RIConvFunction.apply(x, w0, w1, bias, desc)``; returns the pooled output with the R'
    axis kept, (N, Cout, R', H, W).  The argmax map is saved for the backward pass."""

    @staticmethod
    def forward(ctx, x, w0, w1, bias, desc: Desc):
        bank = bank_precompute(desc, w0.detach(), None if w1 is None else w1.detach())
        y, am = ri_conv_forward(desc, x.detach(), bank, None if bias is None else bias.detach())
        ctx.desc = desc
        ctx.has_w1 = w1 is not None
        ctx.has_bias = bias is not None
        ctx.save_for_backward(x.detach(), bank, y, am if am is not None else torch.empty(0, device=x.device))
        return y

    @staticmethod
    def backward(ctx, gy):
        x, bank, y, am = ctx.saved_tensors
        dx, dw0, dw1, db = ri_conv_backward(
            ctx.desc, x, bank, gy.contiguous(), y, am if am.numel() else None, ctx.needs_input_grad[0],
            ctx.needs_input_grad[1] or ctx.needs_input_grad[2], ctx.has_bias and ctx.needs_input_grad[3])
        return dx, dw0, (dw1 if ctx.has_w1 else None), db, None
