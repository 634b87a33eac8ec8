# round 2 session 2: content-addressed tensor-map store: records stress + per-launch determinism probe
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/stress.txt gpurun_out/race.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
echo "== store $rep" >> gpurun_out/stress.txt; timeout 900 python scripts/stress_records.py 24 >> gpurun_out/stress.txt 2>&1
done
timeout 900 python scripts/race_probe.py 30 > gpurun_out/race.txt 2>&1; echo race=$? >> gpurun_out/status.txt
