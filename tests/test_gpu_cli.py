"""The GA command-line driver on a B200: a run interrupted after generation 1
and resumed from its checkpoint writes the same generation log and result as
an uninterrupted run."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _ga(out, gens, resume=False):
    cmd = [sys.executable, "-m", "paper_2107_09789_b200", "ga", "--fixture", "c1c2", "--size", "24", "--mode",
           "dimension", "--population", "4", "--generations", str(gens), "--trials", "2", "--out", str(out)]
    if resume:
        cmd.append("--resume")
    subprocess.run(cmd, cwd=ROOT, check=True, timeout=600, env={**__import__("os").environ, "TOBF_HOST_WORKERS": "2"})


def test_ga_cli_resume(tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    _ga(a, 3)
    _ga(b, 1)
    _ga(b, 3, resume=True)
    la = [json.loads(x) for x in (a / "log.jsonl").read_text().splitlines()]
    lb = [json.loads(x) for x in (b / "log.jsonl").read_text().splitlines()]
    key = lambda r: (r["generation"], r["best_reward"], r["survivor_rewards"])  # noqa: E731
    assert [key(r) for r in la] == [key(r) for r in lb]
    ra, rb = json.loads((a / "result.json").read_text()), json.loads((b / "result.json").read_text())
    assert ra["best_genome"] == rb["best_genome"] and ra["best_reward"] == rb["best_reward"]
