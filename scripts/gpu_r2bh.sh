# round 2 session 2: folded-BatchNorm cache across a CTA's tiles A/B + parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "conv or execute or paired or bf16" > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for rep in 1 2; do
  for v in sc nosc; do
    lib=paper_2107_09789_b200/libtobf.so; [ $v = nosc ] && lib=scripts/_probe_libs/libtobf_nosc.so
    for prec in fp32 bf16; do
      TOBF_LIB=$lib timeout 300 python scripts/conv_levels.py --prec $prec > gpurun_out/levels_${v}_${prec}_$rep.txt 2>&1
      echo "== $v $prec rep$rep $(grep 'conv launches' gpurun_out/levels_${v}_${prec}_$rep.txt)" >> gpurun_out/variants.txt
    done
  done
done
