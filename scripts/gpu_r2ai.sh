# round 2 session 2: epilogue diagnostics (no output stores / no residual loads / no drain)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base nostg noldg nod; do
  lib=scripts/_probe_libs/libtobf_$v.so; [ $v = base ] && lib=paper_2107_09789_b200/libtobf.so
  TOBF_LIB=$lib timeout 300 python scripts/conv_levels.py --prec fp32 > gpurun_out/levels_${v}.txt 2>&1
  echo "== $v $(grep 'conv launches' gpurun_out/levels_${v}.txt)" >> gpurun_out/variants.txt
done
