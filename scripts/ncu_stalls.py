"""Development aid: per-role warp-stall breakdown of a conv_tc_kernel ncu capture
(source page), roles delimited by the setmaxnreg / UTCHMMA landmarks."""
import csv
import subprocess
import sys


def main(path, launch=0):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    lo = starts[launch]
    hi = starts[launch + 1] if launch + 1 < len(starts) else len(rows)
    hdr, data = rows[lo + 1], rows[lo + 2:hi]
    src = hdr.index("Source")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {h: hdr.index(h) for h in reasons}
    ex = hdr.index("Instructions Executed")
    marks = [i for i, r in enumerate(data) if "USETMAXREG" in r[src]]
    mma = [i for i, r in enumerate(data) if "UTCHMMA" in r[src]]
    bounds = [(0, marks[0], "prologue"), (marks[0], marks[1], "A producer"), (marks[1], marks[2], "control/B"),
              (marks[2], min(mma) - 60, "epilogue+sched"), (min(mma) - 60, len(data), "MMA+tail")]
    f = lambda x: float(x or 0)  # noqa: E731
    tot = sum(f(r[idx[h]]) for r in data for h in reasons)
    for a, b, name in bounds:
        part = {h: sum(f(r[idx[h]]) for r in data[a:b]) for h in reasons}
        s = sum(part.values())
        top = sorted(part.items(), key=lambda t: -t[1])[:6]
        print(f"{name:16s} {s / tot * 100:5.1f}% of samples, {sum(f(r[ex]) for r in data[a:b]):.3g} warp-instr; "
              + ", ".join(f"{k[6:]} {v / max(s, 1) * 100:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
