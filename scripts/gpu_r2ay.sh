# round 2 session 2: per-launch determinism probe of the headline forward (find the racing launch)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/race.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python scripts/race_probe.py 60 > gpurun_out/race.txt 2>&1; echo race=$? >> gpurun_out/status.txt
