"""One line per captured kernel of an `ncu --set full` report (duration, warp instructions, DRAM bytes,
occupancy, registers, issue-slot and DRAM/SM throughput, launch shape).

    python profiles/summarize_ncu.py gpurun_out/full_r02b.ncu-rep "header line" > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

M = {
    "t": "gpu__time_duration.sum", "inst": "smsp__inst_executed.sum", "dram_r": "dram__bytes_read.sum",
    "dram_w": "dram__bytes_write.sum", "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread", "issue": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed", "grid": "launch__grid_size",
    "blk": "launch__block_size",
}


def main(rep, header):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M.values())],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"us": 1e3, "ns": 1.0, "ms": 1e6, "Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}
    print("# " + header)
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        g = {k: r[h.index(v)] if v in h else "" for k, v in M.items()}
        def f(k):
            if g[k] in ("", "n/a"):
                return float("nan")
            return float(g[k].replace(",", "")) * scale.get(units[h.index(M[k])], 1.0)
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("bgs::", "")[:34]
        print(f"{name:34s} t={f('t') / 1e3:9.3f}us inst={f('inst') / 1e6:7.2f}M dram={(f('dram_r') + f('dram_w')) / 1e6:7.1f}MB "
              f"occ={f('occ'):5.1f}% regs={int(f('regs'))} issue={f('issue'):5.1f}% dram%={f('dram_pct'):5.1f} "
              f"sm%={f('sm_pct'):5.1f} grid={int(f('grid'))} blk={int(f('blk'))}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
