# quick GPU check: parity tests + per-cell probe (old vs new lib) + bench
set -x
O=gpurun_out/${1:-q}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $O/pytest_gpu.log
[ -f paper_2006_09616_b200/libdtr_old.so ] && DTR_LIB=$PWD/paper_2006_09616_b200/libdtr_old.so timeout 300 python scripts/probe_cells.py > $O/cells_old.txt 2>&1
timeout 300 python scripts/probe_cells.py > $O/cells_new.txt 2>&1
cat $O/cells_old.txt $O/cells_new.txt
timeout 900 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; echo bench=$?
head -c 3000 $O/bench.json
