"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref/librc_ref.so,
built from /root/reference/proj/include by oracle/Makefile).  Run in the build
container (where the reference exists):  python tests/golden/make_golden.py

Each fixture holds seeded inputs and the reference's outputs:
  tiled_*   : rotconv::tiled_scatter_conv (scatter_conv.hpp:330-368) + MultCounter
  raw_*     : rotconv::scatter_conv_raw_multi (scatter_conv.hpp:151-187)
  slices_*  : unpooled RI output built only from reference primitives,
              slice (b, r) = tiled_scatter_conv(X, rot90_plane^r(K_b))  (P1 convention)
The steerable bases are SPEC-defined (no reference code); they are produced by the
oracle's rco_steer and stored in the fixture so the slices depend only on reference code.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402


def dyadic(rng, shape):
    return (rng.integers(-4, 5, shape) / 4).astype(np.float32)


def main():
    assert O.ref_available(), "oracle/_ref/librc_ref.so missing: run make -C oracle"
    rng = np.random.default_rng(20251208)
    out = {}
    # single-orientation drop-in path, including ragged sizes and K in {1,2,3,5}
    for i, (cin, h, w, cout, k) in enumerate([(3, 5, 7, 4, 3), (4, 8, 8, 6, 3), (2, 1, 9, 3, 3),
                                               (5, 6, 4, 2, 1), (3, 7, 7, 2, 5), (2, 6, 5, 3, 2),
                                               (8, 16, 16, 8, 3)]):
        x = rng.standard_normal((cin, h, w)).astype(np.float32)
        wt = (rng.standard_normal((cout, cin, k, k)) / np.sqrt(cin * k * k)).astype(np.float32)
        y, m, a, _ = O.ref_tiled_scatter_conv(x, wt, tile=(32, 32), workers=1)
        out[f"tiled_{i}_x"], out[f"tiled_{i}_w"], out[f"tiled_{i}_y"] = x, wt, y
        out[f"tiled_{i}_counts"] = np.array([m, a], np.uint64)
        out[f"raw_{i}_y"] = O.ref_scatter_conv_raw_multi(x, wt)
    # RI slices, random and dyadic inputs
    cases = [("p4", 4, 5, 6, 7, 3), ("p4m", 8, 4, 8, 8, 4), ("steer", 8, 6, 8, 8, 5),
             ("steer", 16, 3, 5, 6, 2), ("single", 1, 4, 6, 6, 3)]
    for i, (g, R, cin, h, w, cout) in enumerate(cases):
        for kind in ("rand", "dyadic"):
            if kind == "rand":
                x = rng.standard_normal((cin, h, w)).astype(np.float32)
                w0 = (rng.standard_normal((cout, cin, 3, 3)) / np.sqrt(cin * 9)).astype(np.float32)
                w1 = (rng.standard_normal((cout, cin, 3, 3)) / np.sqrt(cin * 9)).astype(np.float32)
            else:
                x, w0, w1 = dyadic(rng, (cin, h, w)), dyadic(rng, (cout, cin, 3, 3)), dyadic(rng, (cout, cin, 3, 3))
            d = O.Desc(1, cin, h, w, cout, 3, g, R)
            bases = O.build_bases(d, w0, w1)
            key = f"slices_{i}_{kind}"
            out[key + "_meta"] = np.array([list(O.GROUPS).index(g), R, cin, h, w, cout], np.int32)
            out[key + "_x"], out[key + "_w0"], out[key + "_w1"] = x, w0, w1
            out[key + "_bases"] = bases
            out[key + "_f"] = O.ref_ri_slices(d, x, w0, bases)
    path = os.path.join(HERE, "reference_fixtures.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
