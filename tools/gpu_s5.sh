# session 4b: new K3+K4 (deferred slow stack, no grid barrier), closure-cache counters
set -x
mkdir -p gpurun_out/s5
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s5/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s5/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s5/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu > gpurun_out/s5/bench.json 2>gpurun_out/s5/bench.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/s5/bench.json'))
for k in ('roofline_large_pool','roofline_large_pool_4e6'): print(k, round(d[k]['us_per_launch'],2), round(d[k]['frac'],4))
print('value', d['value'], d['ms_per_step'])"
python paper_2006_09616_b200/_build.py --profile > /dev/null 2>&1; echo profbuild=$?
for c in "transformer msps 317 3000" "densenet100 msps 317 3000" "lstm msps 317 3000" "treelstm msps 317 3000" "lstm dtr_eq 317 20000" "lstm dtr 100 20000" "treelstm dtr 100 20000" "resnet32 size 286 0"; do
  timeout 300 python tools/probe_prof_c5.py $c 2>&1 | tail -5
done > gpurun_out/s5/prof.log; cat gpurun_out/s5/prof.log
