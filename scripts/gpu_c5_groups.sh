mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
OUT=gpurun_out/c5_groups.jsonl timeout 1500 python scripts/probe_c5_groups.py size,lru,dtr,dtr_eq > gpurun_out/c5_a.log 2>&1; echo rc=$?
OUT=gpurun_out/c5_groups.jsonl timeout 900 python scripts/probe_c5_groups.py msps > gpurun_out/c5_b.log 2>&1; echo rc=$?
cat gpurun_out/c5_a.log gpurun_out/c5_b.log | tail -40
