for g in 0 32 0 32; do
  SPIN_GEMM_DBG=$g timeout 200 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gdbg', $g, round(d['value']), round(d['config']['draft_us_median']), round(d['config']['verify_step_us_median']))"
done
