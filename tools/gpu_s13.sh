# wide global-state CTA engine (512 threads), shared-memory walk mirror for closure cells
set -x
mkdir -p gpurun_out/s13
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s13/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fulllength" > gpurun_out/s13/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s13/pytest_gpu.log
for h in msps dtr_eq; do for m in transformer treelstm lstm; do
  OUT=gpurun_out/s13/c5_groups.jsonl timeout 400 python tools/probe_c5_groups.py $h $m 2>&1 | tail -1
done; done
OUT=gpurun_out/s13/c5_sweep.jsonl timeout 1200 python tools/probe_c5_sweep.py 2 2>&1 | tail -30
