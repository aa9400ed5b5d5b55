"""Summarise one kernel of an ncu --set full capture into the JSON kept under profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.json "capture command line"
"""
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__block_size", "launch__grid_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "smsp__sass_inst_executed_op_utcmma.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__warps_active.avg.per_cycle_active",
]


def main():
    rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            m[k] = f"{vals[i]} {units[i]}".strip()
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = int(float(vals[i].replace(",", "")))
            except ValueError:
                pass
    top = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    m["pc_sampling_stalls_top"] = top
    json.dump({"kernel": m.get("Kernel Name"), "capture": cmd, "metrics": m}, open(out, "w"), indent=1)
    print(json.dumps(m, indent=1))


if __name__ == "__main__":
    main()
