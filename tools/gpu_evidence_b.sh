# Round evidence, part B: the bench line + launch list at HEAD, compute-sanitizer over
# every kernel, the MSPS cells of the config-5 sweep.  usage: bash tools/gpu_evidence_b.sh TAG
set -x
TAG=${1:-r02b}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 2400 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?; head -c 3000 $O/bench.json; echo
timeout 1200 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_reference.json 2>&1; echo ref=$?
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-extra --no-large-pool --no-cpu > $O/bench_ncu.log 2>&1; echo ncu_launch=$?
bash tools/sanitize.sh $O/sanitize
timeout 1800 python tools/msps_sweep.py > $O/msps_sweep.json 2>&1; echo msps=$?; cat $O/msps_sweep.json
