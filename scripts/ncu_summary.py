"""Summarise an ncu --set full capture (.ncu-rep) into a markdown table of the
numbers DESIGN.md and bench.py's roofline cite, one column per captured
launch, and (with --traffic) update profiles/ncu_traffic.json with each
kernel's DRAM bytes per launch and its shared-memory wavefronts per SM per
clock.

    python scripts/ncu_summary.py gpurun_out/prof_r02.ncu-rep [--traffic TAG]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ROWS = [
    ("duration (ncu, cold cache)", "gpu__time_duration.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("registers / thread", "launch__registers_per_thread"),
    ("dynamic shared memory / block", "launch__shared_mem_per_block_dynamic"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit rate", "lts__t_sector_hit_rate.pct"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("shared wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("shared bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("SM active cycles (avg)", "sm__cycles_active.avg"),
    ("local loads (warp instr.)", "smsp__inst_executed_op_local_ld.sum"),
    ("local stores (warp instr.)", "smsp__inst_executed_op_local_st.sum"),
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    return head, units, data


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    path = sys.argv[1]
    tag = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    head, units, data = load(path)
    col = {n: i for i, n in enumerate(head)}
    names = [r[col["Kernel Name"]].split("(")[0] for r in data]
    print("| metric | " + " | ".join(f"`{n}`" for n in names) + " |")
    print("|---|" + "---:|" * len(names))
    for label, m in ROWS:
        if m not in col:
            continue
        u = units[col[m]]
        print(f"| {label} | " + " | ".join(f"{r[col[m]]} {u}".strip() for r in data) + " |")
    # shared wavefronts per SM per active clock
    if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in col and "sm__cycles_active.avg" in col:
        vals = []
        for r in data:
            wf = num(r[col["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]])
            cyc = num(r[col["sm__cycles_active.avg"]])
            vals.append(wf / 148.0 / cyc if wf and cyc else None)
        print("| shared wavefronts / SM / active clock | " +
              " | ".join(f"{v:.3f}" if v else "" for v in vals) + " |")
    stalls = [n for n in head if n.startswith(STALL) and not n.endswith("_not_issued")]
    tops = []
    for r in data:
        tot = sum(num(r[col[n]]) or 0.0 for n in stalls)
        top = sorted(((num(r[col[n]]) or 0.0, n[len(STALL):]) for n in stalls), reverse=True)[:5]
        tops.append(", ".join(f"{k} {100 * v / tot:.1f}" for v, k in top) if tot else "")
    print("| top stalls (% of samples) | " + " | ".join(tops) + " |")
    if tag:
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        try:
            with open(tf) as f:
                rec = json.load(f)
        except OSError:
            rec = {}
        for r, n in zip(data, names):
            short = n.split("::")[-1].split("<")[0].replace("void ", "").strip()
            rd = num(r[col["dram__bytes_read.sum"]]) or 0.0
            wr = num(r[col["dram__bytes_write.sum"]]) or 0.0
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(units[col["dram__bytes_read.sum"]], 1)
            wr *= scale.get(units[col["dram__bytes_write.sum"]], 1)
            entry = {"dram_bytes_per_launch": int(rd + wr),
                     "duration_ms_ncu": (num(r[col["gpu__time_duration.sum"]]) or 0) *
                     (1e-3 if units[col["gpu__time_duration.sum"]] == "us" else 1e-6
                      if units[col["gpu__time_duration.sum"]] == "ns" else 1),
                     "source": f"profiles/{tag}_ncu_full.md ({os.path.basename(path)}, {n})"}
            wf = num(r[col.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0)] or "")
            cyc = num(r[col.get("sm__cycles_active.avg", 0)] or "")
            if wf and cyc:
                entry["smem_wavefronts_per_sm_clk"] = round(wf / 148.0 / cyc, 4)
            rec[short] = entry
        with open(tf, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
