"""The C-ABI boundary on CPU: the library loads, exports every symbol rotconv_c.h
declares, validates with the reference's messages; the product never touches the oracle."""
import ast
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rotconv_c.h")
PKG = os.path.join(ROOT, "paper_2512_08888_b200")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rc_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("rc_bank_precompute", "rc_ri_conv_forward", "rc_ri_conv_forward_host",
              "rc_tiled_scatter_conv_host", "rc_workspace_size", "rc_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2512_08888_b200 import _lib
    L = _lib.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert L.rc_abi_version() == 3


def test_validation_messages_match_reference():
    import paper_2512_08888_b200 as P
    cases = [
        (P.Desc(1, 1, 1, 1, 1, 2, "p4", 4), "transform_kernel: rotation groups need odd square kernels"),
        (P.Desc(1, 1, 1, 1, 1, 3, "steer", 6), "build_orientation_bank: N must be a multiple of 4"),
        (P.Desc(1, 1, 1, 1, 1, 3, "p4m", 8, "subgroup", 3), "subgroup_pool_max: R not divisible by group_size"),
        (P.Desc(1, 0, 1, 1, 1, 3), "Tensor3: dimensions must be positive"),
        (P.Desc(1, 1, 1, 1, 0, 3), "FilterBank: channel counts must be positive"),
        (P.Desc(1, 1, 1, 1, 1, 3, "p4", 8), "GroupSpec: size must be 4 for p4"),
    ]
    for d, msg in cases:
        with pytest.raises(ValueError, match=re.escape(msg)):
            d.validate()
    P.Desc(0, 3, 5, 5, 2, 3, "p4m", 8, "max").validate()  # empty batch is valid


def test_tiled_host_entry_validates_like_reference():
    """rc_tiled_scatter_conv_host checks in the reference's order (scatter_conv.hpp:339-346)
    before touching the device."""
    from paper_2512_08888_b200 import _lib
    L = _lib.lib()
    z = C.c_void_p(0)
    cases = [((2, 4, 4, 3, 3, 3, 3, 32, 32, 1, 1), "tiled_scatter_conv: channel mismatch"),
             ((2, 4, 4, 3, 2, 3, 5, 32, 32, 1, 1), "tiled_scatter_conv: kernel must be square"),
             ((2, 4, 4, 3, 2, 3, 3, 0, 32, 1, 1), "tiled_scatter_conv: tile dims must be >= 1"),
             ((2, 4, 4, 3, 2, 3, 3, 32, 32, 2, 1), "tiled_scatter_conv: invalid halo"),
             ((2, 4, 4, 3, 2, 3, 3, 32, 32, 1, 0), "tiled_scatter_conv: workers must be >= 1")]
    for (cin, h, w, cout, cinw, kh, kw, th, tw, halo, workers), msg in cases:
        st = L.rc_tiled_scatter_conv_host(z, cin, h, w, z, cout, cinw, kh, kw, th, tw, halo, workers,
                                          0, z, None, None, None, 0, 0)
        assert st == _lib.RC_ERR_INVALID and _lib.last_error() == msg


def test_analytic_counts_and_shards():
    import paper_2512_08888_b200 as P
    d = P.Desc(256, 256, 16, 16, 1024, 3, "steer", 8, "subgroup", 4)
    m, a = d.analytic_counts()
    assert m == 2 * 256 * 16 * 16 * 9 * 256 * 1024          # per base kernel, R-independent
    assert a == 2 * 256 * 2116 * 1024
    assert d.alg_flops() == 2 * m and d.eff_flops() == 4 * d.alg_flops()
    p4 = P.Desc(3, 4, 8, 8, 5, 3, "p4", 4)
    p1 = P.Desc(3, 4, 8, 8, 5, 3, "single", 1)
    assert p4.analytic_counts() == p1.analytic_counts()       # SPEC:282 acceptance 4
    for n, world in [(512, 8), (10, 3), (0, 2), (5, 8)]:
        spans = [P.shard_range(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1
    with pytest.raises(ValueError):
        P.shard_range(4, 2, 2)


def test_kernel_selection():
    import paper_2512_08888_b200 as P
    c3 = dict(n=256, c_in=256, h=16, w=16, c_out=1024, k=3, group="steer", orientations=8,
              pool="subgroup", pool_group=4)
    assert P.Desc(**c3).precision == "auto"
    assert P.Desc(**c3).kernel_name() == "tc_k3w16_bf16x3"
    assert P.Desc(**c3, precision="fp32").kernel_name().startswith("simt_k3")
    assert P.Desc(32, 64, 8, 8, 256, 3).kernel_name() == "tc_k3img8_bf16x3"
    assert P.Desc(32, 64, 8, 8, 256, 3, precision="fp32").kernel_name().startswith("simt_k3")
    assert P.Desc(2, 3, 7, 5, 4, 5, "p4", 4, "max").kernel_name() == "generic"
    assert P.Desc(8, 3, 64, 64, 64, 3, "steer", 8, "subgroup", 4).kernel_name().startswith("simt_k3")


def test_dropin_entry_points_run_the_default_tensor_core_kernels():
    """Every reference-named entry point defaults to precision auto; at the C1 (8x8x64->256,
    R=1) and C3 (16x16x256->1024, steer R=8) shapes that is the tcgen05 kernel."""
    import torch
    import paper_2512_08888_b200 as P
    from paper_2512_08888_b200 import _lib
    x1, w1 = torch.empty(32, 64, 8, 8), torch.empty(256, 64, 3, 3)
    for conv in ("scatter", "raw"):   # tiled_scatter_conv, scatter_conv_multi, scatter_conv_raw_multi
        d, _, _ = P.rotconv._single_desc(x1, w1, conv)
        assert d.kernel_name() == "tc_k3img8_bf16x3", (conv, d.kernel_name())
    d, _, _ = P.rotconv._single_desc(x1, w1, "scatter", "fp32")
    assert d.kernel_name().startswith("simt_k3")
    # RIConv / ri_conv at C3
    layer = P.RIConv(torch.empty(1024, 256, 3, 3), torch.empty(1024, 256, 3, 3))
    assert layer.desc(256, 16, 16).kernel_name() == "tc_k3w16_bf16x3"
    # the C-ABI host drop-in (rc_tiled_scatter_conv_host) builds precision AUTO (0) descs
    cd = _lib.rc_desc(1, 64, 8, 8, 256, 3, 0, 1, 0, 1, 0, 0, 0)
    assert _lib.lib().rc_kernel_name(C.byref(cd)) == b"tc_k3img8_bf16x3"
    cd = _lib.rc_desc(256, 256, 16, 16, 1024, 3, 3, 8, 3, 4, 0, 0, 0)
    assert _lib.lib().rc_kernel_name(C.byref(cd)) == b"tc_k3w16_bf16x3"


def test_kernel_size_bound_is_validated():
    """K > 11 is refused before any table sized for 11x11 taps is touched (all entry points
    validate first); K = 11 is accepted by the generic kernel."""
    import paper_2512_08888_b200 as P
    from paper_2512_08888_b200 import _lib
    for k, group in ((13, "single"), (13, "p4"), (15, "p4m")):
        d = P.Desc(1, 2, 16, 16, 3, k, group, {"single": 1, "p4": 4, "p4m": 8}[group])
        with pytest.raises(_lib.RotconvError, match="kernel size > 11 unsupported"):
            d.validate()
        assert d.bank_bytes() == 0 and d.workspace_bytes() == 0 and d.kernel_name() is None
    assert P.Desc(1, 2, 16, 16, 3, 11, "p4", 4).kernel_name() == "generic"
    z = C.c_void_p(0)
    st = _lib.lib().rc_tiled_scatter_conv_host(z, 2, 16, 16, z, 3, 2, 13, 13, 32, 32, 6, 1, 0, z,
                                               None, None, None, 0, 0)
    assert st == _lib.RC_ERR_UNSUPPORTED and "kernel size > 11" in _lib.last_error()


def test_product_never_imports_the_oracle():
    """Only tests/, smoke() and bench.py's CPU legs may touch oracle/."""
    for f in os.listdir(PKG):
        if not f.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(PKG, f)).read())
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            for n in names:
                assert "oracle" not in n, f"{f} imports {n}"
        assert "librc_oracle" not in open(os.path.join(PKG, f)).read()
    for f in os.listdir(os.path.join(PKG, "csrc")):
        src = re.sub(r"//[^\n]*|/\*.*?\*/", "", open(os.path.join(PKG, "csrc", f)).read(), flags=re.S)
        assert "rc_oracle" not in src and "rotconv_ref" not in src and "rco_" not in src


def test_product_fails_loudly_without_extension(monkeypatch):
    from paper_2512_08888_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/librotconv_b200.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()
