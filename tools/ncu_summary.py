"""Summarise ncu raw-page CSVs (tools/profile.sh) into profiles/<tag>_ncu_<cfg>.md and the
per-stage DRAM traffic table profiles/ncu_traffic.json that bench.py reports as roofline.traffic."""
import csv
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGES = [("k_task_spmv", "wt_spread"), ("k_t2_rows", "t2_rows"), ("k_t2_cols", "t2_cols"), ("k_w_sep", "w_spmv"), ("k_w_pair", "w_spmv"), ("k_pair_sigma", "pair_sigma"),
          ("k_t1_cols", "t1_cols"), ("k_t1_rows", "t1_rows"), ("k_cg_update", "cg_update"), ("k_sb_post", "sb_post"),
          ("k_stencil", "stencil"), ("k_cp_dual", "cp_dual")]


def stage_of(name):
    for k, s in STAGES:
        if k in name:
            return s
    return None


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return float("nan")


def summarise(raw_csv, cfg, tag):
    rows = list(csv.reader(open(raw_csv)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}

    def g(r, k):
        return num(r[col[k]]) if k in col else float("nan")

    out, traffic = [], defaultdict(list)
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        short = re.sub(r"\(.*", "", name).replace("tomo_b200::", "").replace("<unnamed>::", "")
        st = stage_of(name)
        t_us = g(r, "gpu__time_duration.sum") / (1000.0 if units[col["gpu__time_duration.sum"]] == "nsecond" else 1.0)
        rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units[col["dram__bytes_read.sum"]], 1)
        wr *= scale.get(units[col["dram__bytes_write.sum"]], 1)
        stalls = []
        for k, i in col.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                v = num(r[i])
                if v == v and v > 0:
                    stalls.append((v, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1
        out.append((short, st, t_us, rd, wr, (rd + wr) / (t_us * 1e3) if t_us > 0 else float("nan"),
                    g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"), g(r, "launch__registers_per_thread"),
                    g(r, "launch__grid_size"), g(r, "launch__block_size"), g(r, "lts__t_sector_hit_rate.pct"),
                    ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in stalls[:3])))
        if st:
            traffic[st].append(rd + wr)
    md = [f"# ncu `--set full --clock-control none` — {cfg} ({tag})", "",
          "One solver step's kernels from `tools/profile.sh` (cold caches, serialised replays: per-launch times",
          "are longer than in the bench; the bench's live per-stage CUDA-event times are the reference).", "",
          "| kernel | stage | time µs | DRAM rd MB | DRAM wr MB | DRAM GB/s | warps active % | regs | grid | block | L2 hit % | top stalls |",
          "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for o in out:
        md.append(f"| `{o[0]}` | {o[1]} | {o[2]:.1f} | {o[3] / 1e6:.2f} | {o[4] / 1e6:.2f} | {o[5]:.0f} | {o[6]:.1f} | "
                  f"{o[7]:.0f} | {o[8]:.0f} | {o[9]:.0f} | {o[10]:.1f} | {o[11]} |")
    return "\n".join(md) + "\n", {k: int(sum(v) / len(v)) for k, v in traffic.items()}


def launches(csv_path, md_path, title):
    """Per-stage share of a `--metrics gpu__time_duration.sum` launch list."""
    from collections import Counter
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = Counter(), Counter()
    for r in rows[1:]:
        st = stage_of(r[ki])
        if not st:
            continue
        v = num(r[vi])
        v = v / 1000 if r[ui] in ("ns", "nsecond") else v
        tot[st] += v
        cnt[st] += 1
    T = sum(tot.values()) or 1
    lines = [f"# {title}", "",
             "Consecutive launches inside the timed solve (`tools/profile.sh`). Cold-cache, serialised per-launch",
             "times: compare the SHARE of the step with bench.py's live `stage_share_of_step`.", "",
             "| stage | launches | mean µs | share |", "|---|---|---|---|"]
    for st in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"| {st} | {cnt[st]} | {tot[st] / cnt[st]:.2f} | {tot[st] / T:.3f} |")
    open(md_path, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    tj_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tj = json.load(open(tj_path)) if os.path.exists(tj_path) else {}
    for cfg in ("c2", "c3", "c4", "c5"):
        raw = os.path.join(src, f"{tag}_full_{cfg}_raw.csv")
        if not os.path.exists(raw):
            continue
        md, traffic = summarise(raw, cfg, tag)
        open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{cfg}.md"), "w").write(md)
        tj[cfg] = traffic
        print(cfg, traffic)
    json.dump(tj, open(tj_path, "w"), indent=1)
    lc = os.path.join(src, f"{tag}_launches_c2.csv")
    if os.path.exists(lc):
        import shutil
        shutil.copy(lc, os.path.join(ROOT, "profiles", f"{tag}_launches_c2.csv"))
        launches(lc, os.path.join(ROOT, "profiles", f"{tag}_launches_c2_summary.md"),
                 "Launch list of the default bench (c2) — `ncu --metrics gpu__time_duration.sum --clock-control none`")
