# round 2 session 2: A producer part timings (lds / sts) and diagnostic builds (no A stores / no A / no drain)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base nost noa nod; do
  lib=scripts/_probe_libs/libtobf_$v.so; [ $v = base ] && lib=paper_2107_09789_b200/libtobf.so
  TOBF_LIB=$lib timeout 300 python scripts/conv_levels.py --prec fp32 > gpurun_out/levels_${v}.txt 2>&1
  echo "== $v $(grep 'conv launches' gpurun_out/levels_${v}.txt)" >> gpurun_out/variants.txt
done
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 0,1,2,3,4,14,20,22,29,34,38 > gpurun_out/roles_ae.txt 2>&1; echo roles=$? >> gpurun_out/status.txt
