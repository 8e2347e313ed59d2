"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        v = v * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        name = r[ki].split("(")[0].replace("void ", "")
        if "gemm_tc_kernel" in r[ki]:
            name = "gemm_tc_kernel<" + r[ki].split("gemm_tc_kernel<")[1].split(">")[0] + ">"
        agg[name][0] += 1
        agg[name][1] += v
        total += v
    out = [f"total {total/1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        out.append(f"{t/1e3:9.3f} ms {100*t/total:5.1f}%  n={n:4d}  avg={t/n:8.1f} us  {name}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
