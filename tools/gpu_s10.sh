# MSPS critical cells: profile (warp-aggregated counters) and group times
set -x
mkdir -p gpurun_out/s10
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python paper_2006_09616_b200/_build.py --profile > /dev/null 2>&1; echo profbuild=$?
for c in "transformer msps 162 0" "lstm msps 286 60000" "treelstm msps 100 60000" "lstm dtr_eq 317 60000"; do
  timeout 400 python tools/probe_prof_c5.py $c 2>&1 | tail -5
done > gpurun_out/s10/prof.log; cat gpurun_out/s10/prof.log
for m in transformer treelstm lstm; do
  OUT=gpurun_out/s10/c5_groups.jsonl timeout 600 python tools/probe_c5_groups.py msps $m 2>&1 | tail -2
done
