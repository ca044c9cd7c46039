# parity tests + per-cell probe + phase profile (no bench)
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
O=gpurun_out/${1:-q}
mkdir -p $O
[ -z "$NOTEST" ] && timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $O/pytest_gpu.log
timeout 300 python scripts/probe_cells.py > $O/cells_new.txt 2>&1
timeout 300 python scripts/probe_prof2.py > $O/prof.txt 2>&1
cat $O/cells_new.txt $O/prof.txt
