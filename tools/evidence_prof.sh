#!/bin/bash
# Profiling part of tools/evidence.sh (no pytest / bench): launch list of one config-2
# round, ncu --set full of the top kernels, in-graph stamps. Outputs under gpurun_out/.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "round/" --csv --log-file gpurun_out/ev_launches.csv python tools/prof_round.py --graph 0 \
  > gpurun_out/ev_launches.log 2>&1
NCU="ncu --set full --import-source on --clock-control none --nvtx --nvtx-include round/"
timeout 300 $NCU -k regex:gemm_tc_kernel -s 12 -c 4 -o gpurun_out/ev_gemm -f python tools/prof_round.py --graph 0 \
  > gpurun_out/ev_ncu1.log 2>&1
timeout 300 $NCU -k regex:attn_kernel -s 1 -c 1 -o gpurun_out/ev_attn -f python tools/prof_round.py --graph 0 \
  > gpurun_out/ev_ncu2.log 2>&1
timeout 300 $NCU -k regex:dproj_kernel -s 40 -c 4 -o gpurun_out/ev_dproj -f python tools/prof_round.py --graph 0 \
  > gpurun_out/ev_ncu3.log 2>&1
timeout 300 $NCU -k regex:attn_decode_kernel -s 20 -c 1 -o gpurun_out/ev_attn_dec -f python tools/prof_round.py --graph 0 \
  > gpurun_out/ev_ncu4.log 2>&1
timeout 300 $NCU -k regex:"resid_norm|swiglu|qkv_epilogue" -s 6 -c 3 -o gpurun_out/ev_epi -f python tools/prof_round.py --graph 0 \
  > gpurun_out/ev_ncu5.log 2>&1
SPIN_STAMPS=gpurun_out/ev_stamps.csv timeout 300 python tools/prof_round.py --graph 1 > gpurun_out/ev_stamps.log 2>&1
ls -la gpurun_out
