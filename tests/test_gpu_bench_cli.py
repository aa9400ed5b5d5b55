"""SPEC bench_cli on the GPU: record counts, the exact CSV header and its
round trip, the mults invariants, the exit code, and the timed scatter cells pinned to the
CPU oracle (float64) on the same seeded inputs bench_cli generates (tools/bench_cli.py
cell_tensors): normwise <= 1e-4, SPEC's 32-bit tolerance."""
import csv
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "bench_cli.py")
HEADER = "mode,input_size,in_channels,out_channels,orientations,repeats,wall_ms,mults,peak_aux_bytes"


def run_cli(tmp_path, *argv):
    out = tmp_path / "sweep.csv"
    r = subprocess.run([sys.executable, CLI, *argv, "--repeats", "2", "--warmup", "1", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    return r, out


def test_grid_36_records_header_roundtrip(tmp_path):
    """SPEC example: grid {8,16,32} x {4,8} x {4,8} x 3 modes -> 36 records."""
    r, out = run_cli(tmp_path, "--sizes", "8", "16", "32", "--cin", "4", "8", "--cout", "4", "8",
                     "--modes", "scatter", "gather", "im2col_matmul")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = out.read_text().splitlines()
    assert lines[0] == HEADER
    recs = list(csv.DictReader(open(out)))
    assert len(recs) == 36
    for q in recs:
        s, ci, co = int(q["input_size"]), int(q["in_channels"]), int(q["out_channels"])
        assert int(q["mults"]) == 32 * s * s * 9 * ci * co  # H W K^2 Cin Cout per image x batch 32
        assert float(q["wall_ms"]) > 0
    # round trip: the CSV re-parses to the printed records (stdout rows)
    modes = ("scatter,", "gather,", "im2col_matmul,", "group_scatter,", "group_gather,")
    printed = [l for l in r.stdout.splitlines() if l.startswith(modes)]
    assert [",".join(q[h] for h in HEADER.split(",")) for q in recs] == printed


def test_group_mults_invariant(tmp_path):
    """SPEC: group_scatter at R = 4 reports mults == scatter's, group_gather 4x."""
    r, out = run_cli(tmp_path, "--sizes", "8", "--cin", "4", "--cout", "8", "--orientations", "4",
                     "--group", "p4", "--modes", "scatter", "group_scatter", "group_gather")
    assert r.returncode == 0, r.stderr[-2000:]
    m = {q["mode"]: int(q["mults"]) for q in csv.DictReader(open(out))}
    assert m["group_scatter"] == m["scatter"] and m["group_gather"] == 4 * m["scatter"]


def test_infeasible_cell_skipped_and_empty_is_error(tmp_path):
    r, out = run_cli(tmp_path, "--sizes", "2", "--cin", "4", "--cout", "4", "--modes", "scatter")
    assert r.returncode != 0 and "kernel > input" in r.stderr and not out.exists()


@pytest.mark.parametrize("cell", [(8, 64, 256), (16, 16, 512), (4, 128, 256)], ids=str)
def test_timed_scatter_cell_matches_oracle(O, dev, cell):
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_cli
    import paper_2512_08888_b200 as P
    size, cin, cout = cell
    args = bench_cli.parse_args(["--batch", "4", "--precision", "auto"])
    gen = torch.Generator(device="cuda").manual_seed(bench_cli.cell_seed(args, size, cin, cout))
    x, w0, _ = bench_cli.cell_tensors(size, cin, cout, args, gen)
    desc = P.Desc(args.batch, cin, size, size, cout, 3, "single", 1, "none", 1, "scatter", args.precision)
    y, _ = P.ri_conv_forward(desc, x, P.bank_precompute(desc, w0))
    od = O.Desc(args.batch, cin, size, size, cout, 3, "single", 1, "none", 1)
    y_ref, _ = O.ri_forward(od, x.double().cpu().numpy(), w0.double().cpu().numpy(), nthreads=8)
    yy = y.double().cpu().numpy().reshape(y_ref.shape)
    assert np.abs(yy - y_ref).max() / np.abs(y_ref).max() <= 1e-4
