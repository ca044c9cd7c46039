# session 4f: EVQ 1024, state ABI, the config-5 sweep critical cells
set -x
mkdir -p gpurun_out/s9
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s9/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fulllength" > gpurun_out/s9/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s9/pytest_gpu.log
python tools/residency_trace.py 200 gpurun_out/s9/residency_N200_estar_v1 > gpurun_out/s9/residency.log 2>&1; echo resid=$?; cat gpurun_out/s9/residency.log
OUT=gpurun_out/s9/c5_sweep.jsonl timeout 900 python tools/probe_c5_sweep.py 2 2>&1 | tail -30
