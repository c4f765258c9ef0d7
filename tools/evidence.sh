#!/bin/bash
# Full evidence run on one GPU: gpu tests, bench (with CPU baseline), launch list of one
# round, ncu --set full of the top kernels. Outputs under gpurun_out/.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev_pytest.txt
timeout 400 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "round/" --csv --log-file gpurun_out/ev_launches.csv python tools/prof_round.py --graph 0 \
  > gpurun_out/ev_launches.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "round/" \
  -k regex:gemm_tc_kernel -s 232 -c 4 -o gpurun_out/ev_gemm -f python tools/prof_round.py --graph 0 > gpurun_out/ev_ncu1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "round/" \
  -k regex:attn_kernel -s 56 -c 1 -o gpurun_out/ev_attn -f python tools/prof_round.py --graph 0 > gpurun_out/ev_ncu2.log 2>&1
cat gpurun_out/ev_pytest.txt; tail -c 600 gpurun_out/ev_bench.json
