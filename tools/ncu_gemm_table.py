"""Tensor-pipe table of an ncu --set full capture of tools/gemm_time_probe.py
(PROBE_ITERS=1: two launches per shape, warm + timed; the second of each pair is kept)."""
import csv
import subprocess
import sys

path, shapes = sys.argv[1], sys.argv[2].split(",")  # e.g. 645:qkv,645:o,...
out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
c = {n: h.index(n) for n in ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                             "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
                             "l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "launch__grid_size",
                             "launch__cluster_dim_x" if "launch__cluster_dim_x" in h else "launch__grid_size")}
kern = rows[2:][1::2]
print(f"{'shape':14s} {'grid':>5s} {'us':>8s} {'tensor%':>8s} {'L2%':>6s} {'L2->SM TB/s':>12s} {'DRAM MB':>8s}")
for s, r in zip(shapes, kern):
    print(f"{s:14s} {r[c['launch__grid_size']]:>5s} {float(r[c['gpu__time_duration.sum']]):8.1f} "
          f"{float(r[c['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']]):8.1f} "
          f"{float(r[c['lts__throughput.avg.pct_of_peak_sustained_elapsed']]):6.1f} "
          f"{float(r[c['l1tex__m_xbar2l1tex_read_bytes.sum.per_second']]):12.2f} {float(r[c['dram__bytes_read.sum']]):8.1f}")
