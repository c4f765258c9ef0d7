#!/bin/bash
# One GPU round-trip: gpu tests, bench (no cpu baseline), optional ncu of a kernel regex.
#   tools/gpu_check.sh [tests|-] [ncu-regex] [ncu-skip]
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
T=${1:-tests}
if [ "$T" != "-" ]; then
  timeout 400 python -m pytest $T -m gpu -x -q 2>&1 | tail -6
fi
timeout 240 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err || tail -5 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.load(open("gpurun_out/bench.json"))
    c = d["config"]
    print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms/round", round(d["ms_per_step"], 3),
          "verify_us", round(c["verify_step_us_median"]), "draft_us", round(c["draft_us_median"]))
    print("classes", {k: round(v, 3) for k, v in c["per_class_ms_one_round"].items()})
    r = d["roofline"]
    print("gemm", round(r["achieved"]), "GB/s", round(r["frac"], 3), "attn", round(r["attention"]["achieved"]),
          round(r["attention"]["frac"], 3), "us", round(r["attention"]["us_per_launch"], 1))
except Exception as e:
    print("bench parse failed", e)
PY
if [ -n "$2" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "round/" -k "regex:$2" -s ${3:-0} -c ${4:-2} \
    -o gpurun_out/prof -f python tools/prof_round.py --graph 0 > gpurun_out/ncu.log 2>&1
  tail -2 gpurun_out/ncu.log
fi
