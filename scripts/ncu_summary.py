"""Summarise an ncu report (raw page) into a markdown table + per-kernel DRAM traffic JSON.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/<name>.md [config] [profiles/ncu_traffic.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps act %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]

STAGE_OF = {"k_t2_rows": "t2_rows", "k_t2_cols": "t2_cols", "k_w_sep": "w_spmv", "k_w<": "w_spmv",
            "k_wt_tasks": "wt_spread", "k_t1_cols": "t1_cols", "k_t1_rows": "t1_rows", "k_cg_update": "cg_update",
            "k_sb_post": "sb_post", "k_stencil": "stencil"}


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * mult


def main():
    rep, out = sys.argv[1], sys.argv[2]
    cfg = sys.argv[3] if len(sys.argv) > 3 else None
    traffic_path = sys.argv[4] if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu summary: `{os.path.basename(rep)}`", "",
             "| kernel | " + " | ".join(k[1] for k in KEYS) + " | top stalls |",
             "|---|" + "---|" * (len(KEYS) + 1)]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        vals = []
        for k, _ in KEYS:
            i = hdr.index(k)
            vals.append(f"{r[i]} {units[i]}".strip())
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        stalls = ", ".join(f"{h} {v:.1f}" for v, h in sorted(st, reverse=True)[:3])
        lines.append(f"| `{name}` | " + " | ".join(vals) + f" | {stalls} |")
        rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        for key, stage in STAGE_OF.items():
            if name.startswith(key) or key in name:
                traffic[stage] = int(rd + wr)
                break
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if cfg and traffic_path:
        data = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        data[cfg] = traffic
        json.dump(data, open(traffic_path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
