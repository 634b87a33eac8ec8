# round 2 session 2: staging depth with the race-free slot release (A/B)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
  for v in base sd55 sd65 sd64; do
    lib=scripts/_probe_libs/libtobf_$v.so; [ $v = base ] && lib=paper_2107_09789_b200/libtobf.so
    for prec in fp32 bf16; do
      TOBF_LIB=$lib timeout 300 python scripts/conv_levels.py --prec $prec > gpurun_out/levels_${v}_${prec}_$rep.txt 2>&1
      echo "== $v $prec rep$rep $(grep 'conv launches' gpurun_out/levels_${v}_${prec}_$rep.txt)" >> gpurun_out/variants.txt
    done
  done
done
