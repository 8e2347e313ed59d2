"""Per-probe ncu evidence from the capture of tools/profile_probes.py
(gpurun_out/ncu_probes.ncu-rep + gpurun_out/probe_order.json): for every
bench probe, the same launch bench.py times, writes
  profiles/<tag>_ncu_<probe>.txt   one-screen summary (tools/ncu_brief.py keys)
  profiles/traffic.json            {probe: dram read+write bytes per launch,
                                    probe_smem: shared-memory bytes, ncu duration,
                                    achieved DRAM GB/s, tensor pipe %}
Multi-launch probes (e.g. decode_hyper = hyper lane init + decode) get one
row per launch; the last launch carries the probe's name."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_brief import KEYS  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return hdr, units, r[2:]


def val(hdr, units, row, key):
    i = hdr.index(key)
    return float(row[i].replace(",", "")) * SCALE.get(units[i], 1.0)


def main(tag):
    rep = os.path.join(ROOT, "gpurun_out", "ncu_probes.ncu-rep")
    order = json.load(open(os.path.join(ROOT, "gpurun_out", "probe_order.json")))
    hdr, units, data = rows(rep)
    labels = []
    for name, n, *_ in order:
        labels += [f"{name}_pre{i}" for i in range(n - 1)] + [name]
    if len(labels) != len(data):
        raise SystemExit(f"{len(data)} kernels captured for {len(labels)} probe launches")
    out = {}
    for label, row in zip(labels, data):
        dram = val(hdr, units, row, "dram__bytes_read.sum") + val(hdr, units, row, "dram__bytes_write.sum")
        dur = val(hdr, units, row, "gpu__time_duration.sum")
        smem = float(row[hdr.index("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")].replace(",", "")) * 128.0
        tp = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
        out[label] = dram
        out[label + "_detail"] = {
            "kernel": row[hdr.index("Kernel Name")][:90], "ncu_s": dur, "dram_bytes": dram,
            "dram_GBps": dram / dur / 1e9 if dur else None, "smem_bytes": smem,
            "tensor_pipe_pct": float(row[hdr.index(tp)].replace(",", "")) if tp in hdr else None}
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{label}.txt"), "w") as f:
            f.write(f"{label} | {row[hdr.index('Kernel Name')][:90]}\n")
            f.write("  (tools/profile_probes.py replay of the bench probe; ncu --set full, "
                    "--clock-control none)\n")
            for k, nm in KEYS + [("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts")]:
                if k in hdr:
                    f.write(f"  {nm:24s} {row[hdr.index(k)]:>16s} {units[hdr.index(k)]}\n")
            f.write(f"  {'achieved DRAM':24s} {dram / dur / 1e9 if dur else 0:16.1f} GB/s\n")
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if not k.endswith("_detail")}, indent=0))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
