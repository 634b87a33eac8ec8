# round 2 session 2: drain/epilogue latency (batched TMEM loads, residual prefetch, pipelined epilogue batches) vs the previous tip
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "conv or execute or bf16" > gpurun_out/pytest_conv.log 2>&1; echo pytest_conv=$? >> gpurun_out/status.txt
for rep in 1 2; do
  for v in head new pre3 pre0 grp1; do
    lib=scripts/_probe_libs/libtobf_$v.so; [ $v = new ] && lib=paper_2107_09789_b200/libtobf.so
    for prec in fp32 bf16; do
      TOBF_LIB=$lib timeout 300 python scripts/conv_levels.py --prec $prec > gpurun_out/levels_${v}_${prec}_$rep.txt 2>&1
      echo "== $v $prec rep$rep $(grep 'conv launches' gpurun_out/levels_${v}_${prec}_$rep.txt)" >> gpurun_out/variants.txt
    done
  done
done
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 0,1,2,3,4,14,20,22,29,34,38 > gpurun_out/roles_af.txt 2>&1; echo roles=$? >> gpurun_out/status.txt
