# round 2 session 2: tensor-map ring + vectorised stem preselection: parent link cost, e2e, parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/workers.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "paired or population or execute" > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for w in 14 14; do
  TOBF_HOST_WORKERS=$w timeout 600 python bench.py --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline > gpurun_out/b_w.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_w.json').read().strip().split('\n')[-1])
e=d['e2e']; h=e['host_ms_per_step']; print('workers=$w', d['value'], round(e['value']), round(e['ms_per_step'],2), round(e['per_call']['value']), json.dumps(h))" >> gpurun_out/workers.txt
done
timeout 600 python scripts/race_probe.py 12 > gpurun_out/race_ring.txt 2>&1; echo race=$? >> gpurun_out/status.txt
