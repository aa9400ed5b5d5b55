"""Config C5: the multi-layer RI classifier (paper_2512_08888_b200/stack.py) against the CPU
oracle composed layer by layer (oracle ri_forward per conv; ReLU, 2x2 max pool, global
average pool and the linear head restated in numpy -- they are builder-defined glue, not
reference ops).

Tolerances (normwise max|d logits| / max|logits| and per-layer output):
  fp32 (CUDA-core kernels everywhere)                       <= 1e-5
  auto (bf16x3 tensor cores where they cover the shape)     <= 2e-4 after 6 conv layers
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def oracle_stack(O, stack, x, nthreads=16):
    spec = stack.spec
    cur = x.astype(np.float32)
    n = cur.shape[0]
    for layer in stack.layers:
        w0 = layer.w0.cpu().numpy()
        w1 = layer.w1.cpu().numpy() if layer.w1 is not None else None
        b = layer.bias.cpu().numpy()
        if layer.kind == "ri":
            d = O.Desc(n, layer.cin, layer.size, layer.size, layer.cout, 3, "steer", spec.orientations,
                       "subgroup", spec.pool_group)
        else:
            d = O.Desc(n, layer.cin, layer.size, layer.size, layer.cout, 3, "single", 1, "none", 1)
        y, _ = O.ri_forward(d, cur, w0, w1, b, nthreads=nthreads)
        y = np.maximum(y.reshape(n, -1, layer.size, layer.size), 0).astype(np.float32)
        if layer.kind == "conv":
            s = layer.size
            y = y.reshape(n, layer.cout, s // 2, 2, s // 2, 2).max(axis=(3, 5))
        cur = np.ascontiguousarray(y, dtype=np.float32)
    feat = cur.mean(axis=(2, 3), dtype=np.float64)
    return feat @ stack.head_w.cpu().numpy().astype(np.float64).T + stack.head_b.cpu().numpy()


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("auto", 2e-4)])
def test_stack_matches_oracle(O, dev, precision, tol):
    from paper_2512_08888_b200.stack import RIStack, StackSpec
    spec = StackSpec(size=32, widths=(32, 64, 128), precision=precision)
    stack = RIStack(spec, dev, seed=3)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (2, 3, 32, 32)).astype(np.float32)
    logits = stack.forward(torch.from_numpy(x).to(dev)).cpu().numpy()
    ref = oracle_stack(O, stack, x)
    err = np.abs(logits - ref).max() / np.abs(ref).max()
    assert err <= tol, f"{precision}: normwise {err:.3e} ({stack.kernels(2)})"


def test_stack_c5_shape_graph_and_kernels(O, dev):
    """The C5 shape (64x64, widths 64/128/256) on 2 images: tensor-core kernels where W is
    16/32, graph replay == eager, finite logits, and the oracle within tolerance."""
    from paper_2512_08888_b200.stack import RIStack, StackSpec
    stack = RIStack(StackSpec(), dev, seed=5)
    ks = stack.kernels(2)
    assert ks[2].startswith("tc_k3strip") and ks[4].startswith("tc_k3w16"), ks
    x = torch.rand((2, 3, 64, 64), device=dev) * 2 - 1
    eager = stack.forward(x).clone()
    graph = stack.graph_forward(x).clone()
    assert torch.equal(eager, graph)
    ref = oracle_stack(O, stack, x.cpu().numpy())
    err = np.abs(eager.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 2e-4, err
