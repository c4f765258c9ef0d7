"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv): per kernel, launches, total / average time, share, DRAM bytes per launch."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    per = collections.defaultdict(lambda: {"n": set(), "t": 0.0, "b": 0.0})
    for r in rows:
        name = r["Kernel Name"]
        name = name.replace("(anonymous namespace)::", "").replace("spin::", "").replace("void ", "").split("(")[0]
        k = per[name]
        k["n"].add(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            k["t"] += v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[unit]
        else:
            k["b"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}[unit]
    total = sum(k["t"] for k in per.values())
    n_all = sum(len(k["n"]) for k in per.values())
    print(f"total {total:.1f} us, {n_all} launches")
    for name, k in sorted(per.items(), key=lambda x: -x[1]["t"]):
        n = len(k["n"])
        print(f"{name[:44]:44s} n={n:4d} total={k['t']:9.1f}us share={100 * k['t'] / total:5.1f}% "
              f"avg={k['t'] / n:7.1f}us dram/launch={k['b'] / n / 1e6:8.2f}MB")


if __name__ == "__main__":
    main(sys.argv[1])
