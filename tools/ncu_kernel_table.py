"""Per-kernel evidence table from one `ncu --set full` report (SURVEY §8d metric list).

usage: python tools/ncu_kernel_table.py report.ncu-rep [n_particles]
Prints, for every captured launch (averaged per kernel name): device time, DRAM bytes and
throughput, L2 / L1 hit rates, L2 reduction / atomic sectors, shared-memory atomics,
executed warp-instructions (and per particle when n is given), lane efficiency (threads
per executed warp-instruction), issue activity and warps active."""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

METRICS = OrderedDict([
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("lts__t_sectors_op_red.sum", "l2_red_sectors"),
    ("lts__t_sectors_op_atom.sum", "l2_atom_sectors"),
    ("smsp__sass_inst_executed_op_shared_atom.sum", "smem_atom_instr"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wf_pct"),
    ("smsp__inst_executed.sum", "warp_instr"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes_per_instr"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
])
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "second": 1e6}


def main():
    rep = sys.argv[1]
    n = float(sys.argv[2]) if len(sys.argv) > 2 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    for m in METRICS:  # section-prefixed names (e.g. "FBSP.TriageCompute.<metric>")
        if m not in col:
            hit = [i for i, h in enumerate(hdr) if h.endswith("." + m)]
            if hit:
                col[m] = hit[0]
    acc = OrderedDict()
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("dpd::", "")
        a = acc.setdefault(name, {"launches": 0})
        a["launches"] += 1
        for m, key in METRICS.items():
            if m not in col:
                continue
            v = r[col[m]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[col[m]]
            if key == "time":
                x *= SCALE.get(u, 1.0)  # -> us
            elif u in SCALE and key.startswith("dram_") and key != "dram_pct":
                x *= SCALE[u]  # -> bytes
            a[key] = a.get(key, 0.0) + x
    print("| kernel | launches | time us | DRAM MB (r+w) | DRAM % peak | L2 hit % | L1 hit % | L2 red sectors | "
          "L2 atom sectors | smem atomics (warp-instr) | smem wavefronts | smem wf % peak | warp-instr | lanes/instr | "
          "issue active % | warps active % |" + (" lane-instr / particle |" if n else ""))
    print("|---" * (16 + (1 if n else 0)) + "|")
    for name, a in acc.items():
        k = a["launches"]
        g = lambda key, d=0.0: a.get(key, d) / k  # noqa: E731
        row = [name, str(k), f"{g('time'):.1f}", f"{(g('dram_read') + g('dram_write')) / 1e6:.1f}",
               f"{g('dram_pct'):.1f}", f"{g('l2_hit_pct'):.1f}", f"{g('l1_hit_pct'):.1f}",
               f"{g('l2_red_sectors'):.3g}", f"{g('l2_atom_sectors'):.3g}", f"{g('smem_atom_instr'):.3g}",
               f"{g('smem_wavefronts'):.3g}", f"{g('smem_wf_pct'):.1f}", f"{g('warp_instr'):.3g}", f"{g('lanes_per_instr'):.1f}", f"{g('issue_active_pct'):.1f}",
               f"{g('warps_active_pct'):.1f}"]
        if n:
            row.append(f"{g('warp_instr') * g('lanes_per_instr') / n:.0f}")
        print("| " + " | ".join(row) + " |")


if __name__ == "__main__":
    main()
