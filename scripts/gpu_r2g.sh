# round 2, call G: scheduler rework (batched claims, smem problem table) + LSTM single-buffer rb kernel
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
rm -f gpurun_out/levels.txt
for args in "--prec fp32" "--prec bf16"; do
  echo "== $args" >> gpurun_out/levels.txt
  timeout 300 python scripts/conv_levels.py $args --order >> gpurun_out/levels.txt 2>&1
done
bash scripts/build_prof_lib.sh > gpurun_out/prof_build.log 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 0,1,3,20,34 > gpurun_out/roles.txt 2>&1; echo roles=$? >> gpurun_out/status.txt
for v in rb4 rb8; do echo "== $v" >> gpurun_out/cfg5.txt; TOBF_LSTM_VARIANT=$v timeout 300 python scripts/cfg5_lstm.py >> gpurun_out/cfg5.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k cfg5 > gpurun_out/pytest_cfg5.log 2>&1; echo cfg5=$? >> gpurun_out/status.txt
