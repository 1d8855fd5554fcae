#!/usr/bin/env bash
# Mirror-pair path check: its own tests first, then the whole GPU suite, then quick bench lines.
timeout 900 python -m pytest tests/test_gpu_sym.py -x -q -s -p no:cacheprovider > gpurun_out/sym_tests.log 2>&1; echo "sym rc=$?" >> gpurun_out/sym_tests.log
tail -5 gpurun_out/sym_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
tail -15 gpurun_out/gputests.log
for c in ${CFGS:-c5 c1 c2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/chk_$c.json 2> gpurun_out/chk_$c.err; echo "$c rc=$?"
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/chk_$c.json").read().strip().splitlines()[-1])
    print("$c", round(d["value"], 2), d["unit"], "e2e", round(d["e2e"]["value"], 2), {k: round(v * 1e3, 2) for k, v in d["roofline"]["stage_ms"].items()}, d["roofline"].get("apply", {}).get("frac"))
except Exception as e:
    print("$c: no line", e)
PY
done
