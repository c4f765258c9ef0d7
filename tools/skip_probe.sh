# timing experiments on the draft projections (results invalid; timing only)
for m in 0; do
  SPIN_DPROJ_DBG=$m SPIN_STAMPS=gpurun_out/stamps_$m.csv timeout 300 python tools/prof_round.py --graph 1 > /dev/null 2>&1
  echo "dbg $m"; python tools/stamps.py gpurun_out/stamps_$m.csv 0 0 2>/dev/null | tail -5
done
