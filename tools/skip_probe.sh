for st in 8 5 4; do
  SPIN_GEMM_STAGES=$st timeout 200 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stages', $st, round(d['value']), round(d['config']['verify_step_us_median']), round(d['roofline']['achieved']))"
done
