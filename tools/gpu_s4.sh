# round-2 session 4: tests, bench-cell split, uncapped config-5 MSPS groups
set -x
mkdir -p gpurun_out/s4
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s4/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s4/pytest_gpu.log
timeout 120 python tools/probe_bench_cells.py > gpurun_out/s4/bench_cells.log 2>&1; cat gpurun_out/s4/bench_cells.log
for m in resnet32 densenet100 unet transformer treelstm lstm; do
  OUT=gpurun_out/s4/c5_msps.jsonl timeout 300 python tools/probe_c5_groups.py msps $m 2>&1 | tail -1
done
