# session check: GPU parity tests, then config-5 heavy groups (h_DTR, h_DTR_eq) and MSPS on the small logs
mkdir -p gpurun_out/s1
O=gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 $O/pytest_gpu.log
OUT=$O/c5_groups.jsonl timeout 900 python scripts/probe_c5_groups.py dtr,dtr_eq transformer,treelstm,lstm,densenet100 > $O/c5.log 2>&1; echo c5=$?
cat $O/c5.log
