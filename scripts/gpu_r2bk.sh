# round 2 session 2: e2e with the parent's torch intra-op pool sized to the cores the workers leave
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/workers.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in 14 12 14 15; do
  TOBF_HOST_WORKERS=$w timeout 600 python bench.py --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline > gpurun_out/b_w.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_w.json').read().strip().split('\n')[-1])
e=d['e2e']; h=e['host_ms_per_step']; print('workers=$w', d['value'], round(e['value']), round(e['ms_per_step'],2), round(e['per_call']['value']), h.get('wait_workers'), h.get('lower_pack'), h.get('link_rows'), h.get('total'))" >> gpurun_out/workers.txt
done
