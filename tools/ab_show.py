"""Summarise tools/ab_run.sh outputs: value, e2e and the per-stage live times."""
import glob, json, sys
pat = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_*.json"
for f in sorted(glob.glob(pat)):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    st = d.get("roofline", {}).get("stage_ms", {})
    print(f"{f.split('/')[-1]:28s} {d['value']:10.1f} e2e {d.get('e2e',{}).get('value',0):10.1f} "
          + " ".join(f"{k}={v*1e3:.1f}" for k, v in st.items()))
