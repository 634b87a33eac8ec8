"""The bench's LER sweep launch (10^7 pairs, RN18 L*), once, for an ncu
instruction-count capture; prints the token count. Writes
profiles/ler_instr.json from an ncu CSV when given --from-csv."""
import argparse
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--from-csv", type=Path)
ap.add_argument("--tokens", type=int)
a = ap.parse_args()
if a.from_csv:
    rows = [r for r in csv.DictReader(l for l in open(a.from_csv) if l.startswith('"'))]
    inst = [float(r["Metric Value"].replace(",", "")) for r in rows if r["Metric Name"] == "smsp__inst_executed.sum"]
    out = {"warp_instr_per_token": inst[-1] / a.tokens, "warp_instr": inst[-1], "tokens": a.tokens,
           "source": "ncu --metrics smsp__inst_executed.sum of the bench's LER sweep launch (scripts/ler_instr.py)"}
    (ROOT / "profiles" / "ler_instr.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)
    sys.exit(0)
import torch  # noqa: E402
from paper_2107_09789_b200 import attacker, fixtures  # noqa: E402
from paper_2107_09789_b200.engine import device  # noqa: E402
from paper_2107_09789_b200.ir import label_sequence  # noqa: E402
ctx = device()
dev = ctx.device
truth = attacker.encode_labels(label_sequence(fixtures.resnet18()))
gen = torch.Generator(device=dev)
gen.manual_seed(0)
B, t_max = 10_000_000, 176
lens = torch.randint(119, 170, (B,), generator=gen, device=dev, dtype=torch.int32)
toks = torch.randint(1, 5, (B, t_max), generator=gen, device=dev, dtype=torch.int8)
attacker.edit_distances(toks, lens, torch.from_numpy(truth).to(dev))
torch.cuda.synchronize()
print("tokens", int(lens.sum().item()))
