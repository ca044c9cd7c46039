# final: every GPU test at HEAD (path halving, the 1e6 pool_argmin check) and the bench line
set -x
O=gpurun_out/r02c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q --durations=8 > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -12 $O/pytest_gpu.log
timeout 2400 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?; head -c 2500 $O/bench.json; echo
