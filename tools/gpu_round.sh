# One GPU session for the round's evidence: smoke, tests, bench, launch list,
# ncu --set full of the top kernels (run under gpurun).  usage: bash tools/gpu_round.sh TAG
set -x
TAG=${1:-s2}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
[ -z "$NOTEST" ] && { timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 $O/pytest_gpu.log; }
[ -z "$NOBENCH" ] && { timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?; head -c 6000 $O/bench.json; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-extra --no-large-pool --no-cpu > $O/bench_ncu.log 2>&1; echo ncu_launch=$?
for n in 1000000 4000000; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_argmin -s 2 -c 1 -o $O/pa_full_$n \
      python tools/pool_argmin_one.py $n 0 > $O/ncu_pa_$n.log 2>&1; echo ncu_pa_$n=$?
  ncu -i $O/pa_full_$n.ncu-rep --page raw --csv > $O/pa_raw_$n.csv 2>/dev/null
  ncu -i $O/pa_full_$n.ncu-rep --page details --csv > $O/pa_details_$n.csv 2>/dev/null
  ncu -i $O/pa_full_$n.ncu-rep --page source --csv --print-source sass > $O/pa_source_sass_$n.csv 2>/dev/null
  rm -f $O/pa_full_$n.ncu-rep        # gpurun copies back <= 64 MiB
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cta_engine -s 3 -c 1 -o $O/cta_full \
    python bench.py --steps 1 --warmup 3 --no-extra --no-large-pool --no-cpu > $O/ncu_cta.log 2>&1; echo ncu_cta=$?
ncu -i $O/cta_full.ncu-rep --page raw --csv > $O/cta_raw.csv 2>/dev/null
ncu -i $O/cta_full.ncu-rep --page details --csv > $O/cta_details.csv 2>/dev/null
rm -f $O/cta_full.ncu-rep
ls -la $O
