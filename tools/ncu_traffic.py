"""Per-kernel DRAM traffic per launch from one `ncu --set full` report -> JSON for bench.py.

usage: python tools/ncu_traffic.py report.ncu-rep out.json workload n_local
Maps kernel names to bench keys (force, bin, scan, scatter) and records
dram__bytes_read.sum + dram__bytes_write.sum, gpu__time_duration.sum, shared-memory
wavefronts and executed warp-instructions per launch
(averaged over the captured launches of that kernel)."""
import csv
import io
import json
import subprocess
import sys

KEYS = {"k_force_tile": "force", "k_force_cells": "force", "k_force_ref": "force", "k_bin": "bin",
        "k_scan": "scan", "k_scatter": "scatter"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in data:
        name = r[col["Kernel Name"]]
        key = next((v for k, v in KEYS.items() if name.startswith("void dpd::" + k) or k in name.split("<")[0]),
                   None)
        if key is None:
            continue
        vals = {}
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"):
            vals[m] = float(r[col[m]].replace(",", "")) * UNIT.get(units[col[m]], 1.0)
        a = acc.setdefault(key, {"launches": 0, "bytes": 0.0, "read": 0.0, "write": 0.0, "time_s": 0.0,
                                 "wf": 0.0, "instr": 0.0, "kernel": name.split("(")[0]})
        a["wf"] += vals["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
        a["instr"] += vals["smsp__inst_executed.sum"]
        a["launches"] += 1
        a["read"] += vals["dram__bytes_read.sum"]
        a["write"] += vals["dram__bytes_write.sum"]
        a["bytes"] += vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
        a["time_s"] += vals["gpu__time_duration.sum"]
    res = {"source": rep.split("/")[-1], "per_launch": {}}
    for k, a in acc.items():
        n = a["launches"]
        res["per_launch"][k] = {"kernel": a["kernel"], "dram_bytes": a["bytes"] / n, "dram_read": a["read"] / n,
                                "dram_write": a["write"] / n, "ncu_time_us": 1e6 * a["time_s"] / n,
                                "smem_wavefronts": a["wf"] / n, "warp_instr": a["instr"] / n,
                                "launches_captured": n, "workload": sys.argv[3], "n_local": int(sys.argv[4])}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
