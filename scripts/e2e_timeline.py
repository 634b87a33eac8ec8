"""Timeline of one end-to-end evaluate_records call (host phases per
micro-batch + device busy spans), to see where the pipeline stalls.
usage: python scripts/e2e_timeline.py [pop] [micro e.g. auto or 8,64]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import population_plans  # noqa: E402
from paper_2107_09789_b200 import fixtures  # noqa: E402
from paper_2107_09789_b200.engine import device  # noqa: E402
from paper_2107_09789_b200.evaluate import Evaluator, PopulationEvaluator  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 256
micro = sys.argv[2] if len(sys.argv) > 2 else "auto"
micro = micro if micro == "auto" else [int(x) for x in micro.split(",")]
ctx = device(0)
g = fixtures.resnet18()
pe = PopulationEvaluator(g, Evaluator(), budget=0.02, trials=8, seed=0, memo={})
plans = population_plans(g, P * 6, 1)
log = []
T0 = [0.0]


def stamp(name):
    log.append((name, 1e3 * (time.perf_counter() - T0[0])))


def wrap(meth, name):
    f = getattr(pe, meth)

    def w(*a, **k):
        stamp(name + ">")
        r = f(*a, **k)
        stamp(name + "<")
        return r
    setattr(pe, meth, w)


for m, n in (("prepare_encoded", "prep"), ("run_attack", "attack"), ("link_forward", "link"),
             ("run_forward", "fwd"), ("collect", "collect")):
    wrap(m, n)
dev_events = []
rf = pe.run_forward


def run_forward(prep, att, *a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = rf(prep, att, *a, **k)
    e1.record()
    dev_events.append((len(prep["cands"]), e0, e1))
    return r


pe.run_forward = run_forward
recv_first = {}
rcv = pe.receive


def receive(result, tables=None):
    c = result[0]
    if c % 8 == 0:
        stamp(f"recv{c}")
    return rcv(result, tables)


pe.receive = receive
for s in range(4):
    ctx.clear_cache()
    log.clear()
    dev_events.clear()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    T0[0] = time.perf_counter()
    pe.evaluate_records(plans[s * P:(s + 1) * P], micro=micro, memo={})
    total = 1e3 * (time.perf_counter() - T0[0])
torch.cuda.synchronize()
print(f"P={P} micro={micro} total {total:.1f} ms")
for name, t in log:
    print(f"  {t:8.2f} {name}")
for n, e0, e1 in dev_events:
    print(f"  device fwd batch of {n}: launch-stream span {start.elapsed_time(e0):8.2f} -> {start.elapsed_time(e1):8.2f}")
print({k: round(v, 2) for k, v in pe.last_host_ms.items()})
pe.close()
