"""Writes profiles/traffic.json (dram__bytes_read.sum + dram__bytes_write.sum
per launch) and a one-screen summary per report, from the ncu --set full
captures taken by tools/gpu_round.sh (gpurun_out/ncu_<probe>.ncu-rep)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        tot += float(vals[i].replace(",", "")) * UNIT.get(units[i], 1)
    return tot


def smem_bytes(rep):
    """Shared-memory wavefronts x 128 B and the kernel duration (ns)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    wf = float(vals[hdr.index("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")].replace(",", ""))
    i = hdr.index("gpu__time_duration.sum")
    dur = float(vals[i].replace(",", "")) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6}.get(units[i], 1)
    return wf * 128.0, dur


def main(tag):
    d = {}
    for probe in ("ctx_attn", "ctx_ffn_gu", "step_attn", "step_wq"):
        rep = os.path.join(ROOT, "gpurun_out", f"ncu_{probe}.ncu-rep")
        if os.path.exists(rep):
            d[probe] = dram_bytes(rep)
            if "attn" in probe:  # the attention kernels' binding resource is shared memory
                b, ns = smem_bytes(rep)
                d[probe + "_smem"] = {"bytes": b, "ncu_ns": ns}
            summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_brief.py"), rep],
                                  capture_output=True, text=True).stdout
            open(os.path.join(ROOT, "profiles", f"{tag}_ncu_{probe}.txt"), "w").write(summ)
    json.dump(d, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
