# timing experiments: skip target-forward kernels (results invalid; timing only)
for m in 0 4; do
  SPIN_VERIFY_SKIP=$m timeout 200 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('vskip', $m, round(d['value']), round(d['config']['draft_us_median']), round(d['config']['verify_step_us_median']))"
done
