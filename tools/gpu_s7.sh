# session 4d: branch-and-bound score passes (pass-1 best prunes slow / stale candidates), LDG addressing
set -x
mkdir -p gpurun_out/s7
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s7/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fulllength" > gpurun_out/s7/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s7/pytest_gpu.log
python paper_2006_09616_b200/_build.py --profile > /dev/null 2>&1; echo profbuild=$?
for c in "transformer msps 317 3000" "densenet100 msps 317 3000" "lstm msps 317 3000" "treelstm msps 317 3000" "lstm dtr_eq 317 20000" "lstm dtr 100 20000" "treelstm dtr 100 20000"; do
  timeout 300 python tools/probe_prof_c5.py $c 2>&1 | tail -4
done > gpurun_out/s7/prof.log; cat gpurun_out/s7/prof.log
for m in transformer treelstm lstm densenet100; do
  OUT=gpurun_out/s7/c5_groups.jsonl timeout 300 python tools/probe_c5_groups.py dtr,dtr_eq,msps $m 2>&1 | tail -3
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu > /dev/null 2>gpurun_out/s7/bench.err; echo bench=$?
timeout 1500 python -m pytest tests/test_gpu_fulllength.py -x -q -s --durations=5 > gpurun_out/s7/pytest_full.log 2>&1; echo pytest_full=$?; tail -8 gpurun_out/s7/pytest_full.log
