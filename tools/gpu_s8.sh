# session 4e: stacked slow/stale candidates (no re-scan), team-bound pruning
set -x
mkdir -p gpurun_out/s8
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s8/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fulllength" > gpurun_out/s8/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s8/pytest_gpu.log
python paper_2006_09616_b200/_build.py --profile > /dev/null 2>&1; echo profbuild=$?
for c in "transformer msps 317 40000" "treelstm msps 317 20000" "lstm msps 317 20000" "lstm dtr_eq 317 20000" "lstm dtr 100 20000"; do
  timeout 200 python tools/probe_prof_c5.py $c 2>&1 | tail -4
done > gpurun_out/s8/prof.log; cat gpurun_out/s8/prof.log
for m in transformer treelstm lstm; do
  OUT=gpurun_out/s8/c5_groups.jsonl timeout 240 python tools/probe_c5_groups.py msps,dtr_eq $m 2>&1 | tail -3
done
