"""Summarise an ncu report (raw page) into the markdown kept under profiles/.

usage: python scripts/ncu_summary.py gpurun_out/x.ncu-rep "title" > profiles/x.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("Kernel Name", "kernel"),
    ("Grid Size", "grid"),
    ("Block Size", "block"),
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def main(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    print(f"# {title}\n\nSource: `{path}` (ncu --set full --clock-control none)\n")
    for n, r in enumerate(data):
        print(f"## launch {n}\n\n| metric | value |\n|---|---|")
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                print(f"| {label} | {r[i]} {units[i]} |")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(stalls, reverse=True)[:6])
        print(f"| top stall reasons (sampled) | {top} |\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
