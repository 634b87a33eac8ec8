# round 2, call U: epilogue U=16 rows per batch for <=1 operand chains
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/levels.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for args in "--prec fp32" "--prec bf16" "--fixture vgg16 --mode dimension --pop 8 --prec bf16"; do
  echo "== $args" >> gpurun_out/levels.txt
  timeout 300 python scripts/conv_levels.py $args --order 2>&1 | head -60 >> gpurun_out/levels.txt
done
bash scripts/build_prof_lib.sh > gpurun_out/prof_build.log 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 1,4,20,34 > gpurun_out/roles.txt 2>&1
