# final at HEAD: every GPU test, then the bounds-checked build over every kernel
set -x
O=gpurun_out/r02d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; cat $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q --durations=5 > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -8 $O/pytest_gpu.log
bash tools/bounds_check.sh $O/bounds
