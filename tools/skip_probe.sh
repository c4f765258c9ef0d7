for nw in 8 4; do
  SPIN_DPROJ_NW=$nw SPIN_STAMPS=gpurun_out/st_$nw.csv timeout 300 python tools/prof_round.py --graph 1 > /dev/null 2>&1
  echo "nw $nw"; python tools/stamps.py gpurun_out/st_$nw.csv 0 0 2>/dev/null | grep -v attn | tail -4
  SPIN_DPROJ_NW=$nw timeout 200 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['config']['draft_us_median']))"
done
