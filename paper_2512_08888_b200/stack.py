"""Multi-layer rotation-invariant classifier forward (config C5).

The paper's base block replaces the first convolution of every U-Net block with the RI
conv and pools "across every four symmetric rotations"; the second
convolution of the block stays a standard one (SPEC train_demo MicroNet).
ReLU, the 2x2 down-sampling and the head are not specified anywhere in the reference; the
stack below is builder-defined:

    input  (N, 3, 64, 64)
    block1 RI steer R=8, 3 -> 64, subgroup-4 max (-> 128 ch) + bias + ReLU   @64x64
           conv R=1 128 -> 64 + bias + ReLU                                  @64x64
           maxpool 2x2                                                       -> 32x32
    block2 RI 64 -> 128 (-> 256 ch) + ReLU; conv 256 -> 128 + ReLU; pool    -> 16x16
    block3 RI 128 -> 256 (-> 512 ch) + ReLU; conv 512 -> 256 + ReLU; pool   -> 8x8
    head   global average pool + linear 256 -> 10

Every conv is one fused launch of the C-ABI (rc_ri_conv_forward, bias and ReLU in the
epilogue); the glue is rc_maxpool2x2 / rc_gap_linear.  Weights are random-init (no
checkpoints exist); the whole forward can be captured in a CUDA graph.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import check, lib
from .rotconv import Desc, _ptr, _stream, bank_precompute, ri_conv_forward


@dataclass
class StackSpec:
    in_channels: int = 3
    size: int = 64
    widths: tuple = (64, 128, 256)
    orientations: int = 8          # steerable N (B = N/4 bases)
    pool_group: int = 4            # subgroup-4 max pooling
    classes: int = 10
    precision: str = "auto"        # tcgen05 bf16x3 where the kernel covers the shape, else FP32


@dataclass
class _Layer:
    kind: str                      # "ri" | "conv"
    cin: int
    cout: int
    size: int
    w0: torch.Tensor
    w1: torch.Tensor | None
    bias: torch.Tensor
    banks: dict = field(default_factory=dict)

    def desc(self, n: int, spec: StackSpec) -> Desc:
        if self.kind == "ri":
            return Desc(n, self.cin, self.size, self.size, self.cout, 3, "steer", spec.orientations,
                        "subgroup", spec.pool_group, "scatter", spec.precision, "relu")
        return Desc(n, self.cin, self.size, self.size, self.cout, 3, "single", 1, "none", 1,
                    "scatter", spec.precision, "relu")

    def out_channels(self, spec: StackSpec) -> int:
        return self.cout * (spec.orientations // spec.pool_group) if self.kind == "ri" else self.cout


class RIStack:
    """The C5 classifier.  ``forward(x)`` takes (N, 3, S, S) float32 CUDA and returns logits."""

    def __init__(self, spec: StackSpec = StackSpec(), device="cuda", seed: int = 0):
        self.spec = spec
        self.device = torch.device(device)
        g = torch.Generator(device=self.device).manual_seed(seed)

        def uni(shape, scale):
            return ((torch.rand(shape, generator=g, device=self.device) * 2 - 1) * scale).contiguous()

        self.layers: list[_Layer] = []
        cin, size = spec.in_channels, spec.size
        for width in spec.widths:
            s = 1 / math.sqrt(cin * 9)
            ri = _Layer("ri", cin, width, size, uni((width, cin, 3, 3), s), uni((width, cin, 3, 3), s),
                        uni((width,), 0.1))
            self.layers.append(ri)
            c2 = ri.out_channels(spec)
            s = 1 / math.sqrt(c2 * 9)
            self.layers.append(_Layer("conv", c2, width, size, uni((width, c2, 3, 3), s), None, uni((width,), 0.1)))
            cin, size = width, size // 2
        self.head_w = uni((spec.classes, cin), 1 / math.sqrt(cin))
        self.head_b = uni((spec.classes,), 0.1)
        self._bufs: dict = {}
        self._graphs: dict = {}

    # ------------------------------------------------------------------ bookkeeping
    def descs(self, n: int) -> list[Desc]:
        return [l.desc(n, self.spec) for l in self.layers]

    def alg_flops(self, n: int) -> int:
        return sum(d.alg_flops() for d in self.descs(n))

    def eff_flops(self, n: int) -> int:
        return sum(d.eff_flops() for d in self.descs(n))

    def kernels(self, n: int) -> list[str]:
        return [d.kernel_name() for d in self.descs(n)]

    def launches_per_forward(self, n: int) -> int:
        convs = sum(2 if k.startswith("tc_") else 1 for k in self.kernels(n))
        return convs + len(self.spec.widths) + 1  # + maxpools + head

    def _bank(self, layer: _Layer, d: Desc):
        key = (d.h, d.w, d.precision)
        if key not in layer.banks:
            layer.banks[key] = bank_precompute(d, layer.w0, layer.w1)
        return layer.banks[key]

    def _buffers(self, n: int):
        if n not in self._bufs:
            outs = []
            for l in self.layers:
                outs.append(torch.empty((n, l.out_channels(self.spec), l.size, l.size), device=self.device))
                if l.kind == "conv":
                    outs.append(torch.empty((n, l.cout, l.size // 2, l.size // 2), device=self.device))
            amaps = [torch.empty((n, l.cout, self.spec.orientations // self.spec.pool_group, l.size, l.size),
                                 dtype=torch.uint8, device=self.device) if l.kind == "ri" else None
                     for l in self.layers]
            logits = torch.empty((n, self.spec.classes), device=self.device)
            self._bufs[n] = (outs, amaps, logits)
        return self._bufs[n]

    # ------------------------------------------------------------------- forward
    def forward(self, x: torch.Tensor, argmax: bool = False) -> torch.Tensor:
        n = x.shape[0]
        if tuple(x.shape[1:]) != (self.spec.in_channels, self.spec.size, self.spec.size):
            raise ValueError("RIStack: input must be (N, in_channels, size, size)")
        outs, amaps, logits = self._buffers(n)
        cur = x.contiguous()
        oi = 0
        L = lib()
        for li, layer in enumerate(self.layers):
            d = layer.desc(n, self.spec)
            y = outs[oi]
            oi += 1
            am = amaps[li] if (argmax or layer.kind == "ri") else None
            ri_conv_forward(d, cur, self._bank(layer, d), layer.bias,
                            out=y.view(n, layer.cout, -1, layer.size, layer.size), argmax=am)
            cur = y
            if layer.kind == "conv":
                p = outs[oi]
                oi += 1
                check(L.rc_maxpool2x2(n, layer.cout, layer.size, layer.size, _ptr(cur), _ptr(p),
                                      _stream(self.device)))
                cur = p
        c, hw = cur.shape[1], cur.shape[2]
        check(L.rc_gap_linear(n, c, hw, hw, _ptr(cur), _ptr(self.head_w), _ptr(self.head_b), self.spec.classes,
                              _ptr(logits), _stream(self.device)))
        return logits

    def graph_forward(self, x: torch.Tensor) -> torch.Tensor:
        """forward() replayed from a CUDA graph captured per input buffer (launch overhead
        of the ~15 launches removed).  x must be the same tensor on every call."""
        key = (x.data_ptr(), x.shape[0])
        if key not in self._graphs:
            s = torch.cuda.Stream(self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                self.forward(x)  # banks, buffers and kernel attributes outside the capture
            torch.cuda.current_stream(self.device).wait_stream(s)
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                out = self.forward(x)
            self._graphs[key] = (g, out)
        g, out = self._graphs[key]
        g.replay()
        return out
