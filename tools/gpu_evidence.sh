# Round evidence, part A: smoke, every GPU test, the bench line and the reference arm,
# the ncu launch list of the bench command, ncu --set full of the top kernels.
# usage: bash tools/gpu_evidence.sh TAG
set -x
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q --durations=12 > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -16 $O/pytest_gpu.log
timeout 2400 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?; head -c 5000 $O/bench.json; echo
timeout 1200 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_reference.json 2>&1; echo ref=$?
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-extra --no-large-pool --no-cpu > $O/bench_ncu.log 2>&1; echo ncu_launch=$?
for n in 1000000 4000000; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_argmin -s 2 -c 1 -o $O/pa_full_$n \
      python tools/pool_argmin_one.py $n 0 > $O/ncu_pa_$n.log 2>&1; echo ncu_pa_$n=$?
  ncu -i $O/pa_full_$n.ncu-rep --page raw --csv > $O/pa_raw_$n.csv 2>/dev/null
  ncu -i $O/pa_full_$n.ncu-rep --page details --csv > $O/pa_details_$n.csv 2>/dev/null
  rm -f $O/pa_full_$n.ncu-rep
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cta_engine_g -s 0 -c 1 -o $O/cta_lstm \
    python tools/one_cell_c5.py lstm dtr_eq 317 20000 1 > $O/ncu_cta_lstm.log 2>&1; echo ncu_cta=$?
ncu -i $O/cta_lstm.ncu-rep --page raw --csv > $O/cta_lstm_raw.csv 2>/dev/null
ncu -i $O/cta_lstm.ncu-rep --page details --csv > $O/cta_lstm_details.csv 2>/dev/null
rm -f $O/cta_lstm.ncu-rep
ls -la $O
