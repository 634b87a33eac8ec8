# round 2, call AB: FADD2 residuals in the A producer's hi/lo split (fp32 + bf16) — timing A/B + parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for v in base fadd2; do
  for prec in fp32 bf16; do
    echo "== $v $prec rep$rep $(TOBF_LIB=scripts/_probe_libs/libtobf_$v.so timeout 300 python scripts/conv_levels.py --prec $prec 2>&1 | grep 'conv launches')" >> gpurun_out/variants.txt
  done
  echo "== $v vgg rep$rep $(TOBF_LIB=scripts/_probe_libs/libtobf_$v.so timeout 300 python scripts/conv_levels.py --fixture vgg16 --mode dimension --pop 8 --prec bf16 2>&1 | grep 'conv launches')" >> gpurun_out/variants.txt
done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
