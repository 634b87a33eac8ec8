"""Fold an ncu metrics capture of one step's conv launches into profiles/conv_traffic.json.

The capture (run on the GPU box, one GPU):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --print-units base -k regex:conv_tc_kernel --launch-skip S -c L --csv \
      --log-file gpurun_out/conv_traffic.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps
where L = conv launches per step and S = L (skip the warm-up step).
usage: python scripts/conv_traffic.py gpurun_out/conv_traffic.csv FLOPS_PER_STEP L
"""
import collections
import csv
import io
import json
import sys
from pathlib import Path


def main(path, flops, launches):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    per = collections.defaultdict(dict)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
    for r in rows:
        per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
    assert len(per) == launches, (len(per), launches)
    rd = sum(v["dram__bytes_read.sum"] for v in per.values())
    wr = sum(v["dram__bytes_write.sum"] for v in per.values())
    ns = sum(v["gpu__time_duration.sum"] for v in per.values())
    out = {"flops_per_step": flops, "conv_launches_per_step": launches, "dram_bytes_per_step": int(rd + wr),
           "dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "ncu_conv_ms_per_step": ns / 1e6,
           "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum over {launches} conv launches of one "
                     "bench step (profiles/conv_traffic.json)"}
    Path("profiles/conv_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
