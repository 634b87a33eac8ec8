# round 2 session 2: tail alignment with split-K decided on the unaligned groups (bit-identical problems) A/B + parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/tail.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TOBF_TAIL_ALIGN=0.5 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_tail.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
for rep in 1 2; do
for f in 0 0.3 0.5 0.7; do
  TOBF_TAIL_ALIGN=$f timeout 600 python bench.py --no-e2e --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline > gpurun_out/b_tail.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_tail.json').read().strip().split('\n')[-1])
print('f=$f rep$rep', d['value'], d['ms_per_step'], d['roofline']['conv_ms_per_step'], d['gpu_launches'])" >> gpurun_out/tail.txt
done
done
