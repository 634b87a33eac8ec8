# round 2 session 3, call AD: e2e alone on a box (no test suite before it), twice; host CPU info
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/e2e_alone.txt
nproc > gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt; uptime >> gpurun_out/host.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do
  timeout 600 python bench.py --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline > gpurun_out/b_e.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_e.json').read().strip().split('\n')[-1])
e=d['e2e']; h=e['host_ms_per_step']; print(round(d['value']), round(e['value']), round(e['ms_per_step'],2), h['trace_prep'], h['receive'], h['wait_workers'], h['total'])" >> gpurun_out/e2e_alone.txt
done
