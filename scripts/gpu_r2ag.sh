# round 2 session 2: input im2col for the stem (1x1 GEMM over a shared im2col matrix, TMA A) vs direct
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
for rep in 1 2; do
  for v in 1 0; do
    for prec in fp32 bf16; do
      TOBF_INPUT_IM2COL=$v timeout 300 python scripts/conv_levels.py --prec $prec > gpurun_out/levels_x${v}_${prec}_$rep.txt 2>&1
      echo "== im2col=$v $prec rep$rep $(grep 'conv launches' gpurun_out/levels_x${v}_${prec}_$rep.txt)" >> gpurun_out/variants.txt
    done
  done
done
