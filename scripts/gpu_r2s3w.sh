# round 2 session 3, call W: e2e steps in flight (2 / 3 / 4) and host workers (14 / 15), alternated
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/e2e_depth.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do
  for cfg in "2 14" "3 14" "4 14" "3 15"; do
    set -- $cfg
    TOBF_HOST_WORKERS=$2 timeout 600 python bench.py --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline --e2e-depth $1 > gpurun_out/b_d.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/b_d.json').read().strip().split('\n')[-1])
e=d['e2e']; print('depth=$1 workers=$2', round(d['value']), round(e['value']), round(e['ms_per_step'],2))" >> gpurun_out/e2e_depth.txt
  done
done
