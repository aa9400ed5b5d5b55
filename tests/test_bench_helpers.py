"""bench.py helpers that shape the JSON contract (CPU only: no kernel is launched)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_smem_traffic_c3_geometry():
    import bench
    import paper_2512_08888_b200 as P
    d = P.Desc(256, 256, 16, 16, 1024, 3, "steer", 8, "subgroup", 4, "scatter", "auto")
    b = bench.smem_traffic(d, "tc_k3w16_bf16x3")
    # carry bands: 4 bands x 2 bases of N = 64 px; K-step = Wh + Wl reads (2 x 4 KB), B rows
    # 128 + 64 (x 32 B), TMA weight writes 2 x 4 KB; X (hi + lo) written once per unit
    per_kstep = 2 * 4096 + 192 * 32 + 2 * 4096
    per_item = 2 * 4 * (9 * 4 * 4 * per_kstep + 2 * 4 * 64 * 128)
    assert b == per_item * 256 * 8
    assert 53e9 < b < 55e9
    assert bench.smem_traffic(d, "simt_k3<8,2,4>") is None
    one = bench.smem_traffic(d, "tc_k3w16_bf16")
    assert one < b / 2  # one pass: 1 A + 1 B read and 1 weight part per K-step


def test_smem_roofline_fields():
    import bench
    import paper_2512_08888_b200 as P
    d = P.Desc(256, 256, 16, 16, 1024, 3, "steer", 8, "subgroup", 4, "scatter", "auto")
    if not d.kernel_name().startswith("tc_"):  # CPU container: the dispatcher answers without a GPU
        assert bench.smem_roofline(d, 2.35) is None or bench.smem_roofline(d, 2.35)["unit"] == "TB/s"
        return
    r = bench.smem_roofline(d, 2.35)
    assert r["unit"] == "TB/s" and abs(r["peak"] - 37.2) < 0.1 and 0.5 < r["frac"] < 0.7


def test_clock_sampler_unsampled_summary():
    import bench
    c = bench.ClockSampler(0)
    s = c.summary()
    assert s["reasons"] == ["unsampled"] and s["samples"] == 0
    c.rows.append((1965.0, 1965.0, ["Not Active", "Not Active", "Not Active", "Active"]))
    s = c.summary()
    assert s["sm_mhz"] == 1965.0 and s["reasons"] == ["sw_power_cap"] and s["samples"] == 1


def test_reference_arm_runs_the_reference_code_on_a_sample():
    """cpu_reference: kind "reference" = R x the unmodified tiled_scatter_conv (oracle/_ref),
    kind "port" = the oracle's reuse loop; both report the sample they timed."""
    import bench
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    wl = (6, 8, 8, 8, 16, 3, "steer", 8, "subgroup", 4, "tiny")
    v, info = bench.cpu_reference(wl, 2, target_s=0.0, kind="reference")
    assert v > 0 and info["images"] == 2 and info["cores"] == 2
    assert info["kind"] == ("reference" if O.ref_available() else "port")
    vp, ip = bench.cpu_reference(wl, 2, target_s=0.0, kind="port", m0=3)
    assert vp > 0 and ip["kind"] == "port" and ip["images"] == 3


def test_both_arms_quote_the_same_config():
    import argparse
    import bench
    for name in ("c1", "c3", "c4"):
        args = argparse.Namespace(workload=name, gpus=2)
        c = bench.workload_config(args, bench.WORKLOADS[name], 2)
        assert c == bench.workload_config(args, bench.WORKLOADS[name], 2)
        assert "kernel" not in c and "precision" not in c
    c4 = bench.workload_config(argparse.Namespace(workload="c4", gpus=8), bench.WORKLOADS["c4"], 8)
    assert c4["global_batch"] == 512 and c4["n_per_gpu"] == 64
