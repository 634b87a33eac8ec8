# round 2, call AA: merged N=128 MMA (a_hi x [b_hi|b_lo]) for BN=64 tf32 — timing A/B + parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for v in base merge; do
  echo "== $v fp32 rep$rep $(TOBF_LIB=scripts/_probe_libs/libtobf_$v.so timeout 300 python scripts/conv_levels.py --prec fp32 2>&1 | grep 'conv launches')" >> gpurun_out/variants.txt
done
done
TOBF_LIB=scripts/_probe_libs/libtobf_merge.so timeout 300 python scripts/conv_levels.py --prec fp32 --order 2>&1 | head -20 >> gpurun_out/variants.txt
TOBF_LIB=scripts/_probe_libs/libtobf_merge.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "conv or execute or population or cfg1 or cfg2 or smoke or micro" > gpurun_out/pytest_merge.log 2>&1; echo merge_parity=$? >> gpurun_out/status.txt
