cd "$GRAFT_REPO_ROOT" || exit 1
for rep in 1 2; do for pf in 99 4 6 8; do
  SPIN_GEMM_STAGES=$pf timeout 300 python bench.py --no-cpu-baseline --no-parity --max-micro-batches 1 > gpurun_out/abst_${pf}_${rep}.json 2> gpurun_out/abst_${pf}_${rep}.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/abst_${pf}_${rep}.json').read().strip().splitlines()[-1]);c=d['config'];print('stages=$pf rep=$rep',round(d['value']),round(c['verify_step_us_median']),round(c['draft_us_median']),round(d['roofline']['us_per_launch'],2),d['clocks']['sm_mhz'])" >> gpurun_out/ab_stages_summary.txt 2>&1
done; done
