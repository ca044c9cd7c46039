# h_DTR_eq lcache bound: parity (all GPU tests incl. full-length) and the LSTM / TreeLSTM groups
set -x
mkdir -p gpurun_out/s14
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s14/smoke.log 2>&1; echo smoke=$?
for m in lstm treelstm transformer; do
  OUT=gpurun_out/s14/c5_groups.jsonl timeout 300 python tools/probe_c5_groups.py dtr_eq,dtr $m 2>&1 | tail -2
done
timeout 2400 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/s14/pytest_gpu.log 2>&1; echo pytest=$?; tail -12 gpurun_out/s14/pytest_gpu.log
