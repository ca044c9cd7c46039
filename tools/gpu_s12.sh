# late-phase MSPS: marginal cost per decision between caps
set -x
mkdir -p gpurun_out/s12
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python paper_2006_09616_b200/_build.py --profile > /dev/null 2>&1; echo profbuild=$?
for c in "transformer msps 162 30000" "transformer msps 162 45000" "treelstm msps 100 40000" "treelstm msps 100 70000"; do
  timeout 300 python tools/probe_prof_c5.py $c 2>&1 | tail -6
done > gpurun_out/s12/prof.log; cat gpurun_out/s12/prof.log
