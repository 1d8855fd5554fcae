import glob, json, os
for f in sorted(glob.glob("gpurun_out/" + (__import__("sys").argv[1] if len(__import__("sys").argv) > 1 else "ab15") + "/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(os.path.basename(f), round(d["value"], 2), r["kernel"], r["frac"], {k: round(v * 1e3, 1) for k, v in r["stage_ms"].items()})
    except Exception as e:
        print(f, "ERR", e)
