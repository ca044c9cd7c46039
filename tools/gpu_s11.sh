# multi-candidate closure walk, multi-source event walk, CTA team for closure heuristics on global state
set -x
mkdir -p gpurun_out/s11
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s11/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fulllength" > gpurun_out/s11/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s11/pytest_gpu.log
python paper_2006_09616_b200/_build.py --profile > /dev/null 2>&1; echo profbuild=$?
for c in "transformer msps 162 20000" "treelstm msps 100 20000" "lstm msps 286 60000"; do
  timeout 300 python tools/probe_prof_c5.py $c 2>&1 | tail -6
done > gpurun_out/s11/prof.log; cat gpurun_out/s11/prof.log
python paper_2006_09616_b200/_build.py > /dev/null 2>&1
for m in transformer treelstm lstm; do
  OUT=gpurun_out/s11/c5_groups.jsonl timeout 400 python tools/probe_c5_groups.py msps $m 2>&1 | tail -2
done
