#!/bin/bash
# A/B of environment settings on the config-2 bench (one GPU):
#   tools/ab.sh "SPIN_X=1" "SPIN_X=2 SPIN_Y=0" ...   (an empty string = defaults)
# prints value / draft / verify per setting; full lines in gpurun_out/ab_<i>.json
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
i=0
for setting in "$@"; do
  env $setting timeout 300 python bench.py --no-cpu-baseline --no-parity --steps ${AB_STEPS:-30} ${AB_ARGS:-} \
    > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python - "$setting" gpurun_out/ab_$i.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    c = d["config"]
    print(f"[{sys.argv[1] or 'default'}] value {d['value']:.0f} e2e {d['e2e']['value']:.0f} ms/step {d['ms_per_step']:.3f} "
          f"verify_us {c.get('verify_step_us_median', 0):.0f} draft_us {c.get('draft_us_median', 0):.0f}")
except Exception as e:
    print(f"[{sys.argv[1]}] failed: {e}")
PY
  i=$((i + 1))
done
