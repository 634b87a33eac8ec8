# round 2 session 2: release the A staging slot once its rows have landed (dependency branch) vs after the split
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/race_land.txt gpurun_out/stress.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python scripts/race_probe.py 40 > gpurun_out/race_land.txt 2>&1; echo race=$? >> gpurun_out/status.txt
echo "== landed" >> gpurun_out/stress.txt; timeout 900 python scripts/stress_records.py 24 >> gpurun_out/stress.txt 2>&1
for rep in 1 2; do
  for v in landed late racy; do
    lib=paper_2107_09789_b200/libtobf.so; [ $v = late ] && lib=scripts/_probe_libs/libtobf_late.so; [ $v = racy ] && lib=scripts/_probe_libs/libtobf_opshead.so
    for prec in fp32 bf16; do
      TOBF_LIB=$lib timeout 300 python scripts/conv_levels.py --prec $prec > gpurun_out/levels_${v}_${prec}_$rep.txt 2>&1
      echo "== $v $prec rep$rep $(grep 'conv launches' gpurun_out/levels_${v}_${prec}_$rep.txt)" >> gpurun_out/variants.txt
    done
  done
done
