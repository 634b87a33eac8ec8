# round 2 session 2: tensor-map acquire fence vs none under the records stress
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/stress.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
echo "== nofence $rep" >> gpurun_out/stress.txt; TOBF_LIB=scripts/_probe_libs/libtobf_nofence.so timeout 900 python scripts/stress_records.py 24 >> gpurun_out/stress.txt 2>&1
echo "== fence $rep" >> gpurun_out/stress.txt; timeout 900 python scripts/stress_records.py 24 >> gpurun_out/stress.txt 2>&1
done
