# Memory-safety check without compute-sanitizer (closed on the GPU pool): a build with
# every state access bounds-checked against the simulation's layout (-DDTR_BOUNDS,
# traps on the first violation), run over every kernel's sanitizer case and the
# quick GPU parity tests.  usage: bash tools/bounds_check.sh OUTDIR
O=${1:-gpurun_out/bounds}
mkdir -p $O
python paper_2006_09616_b200/_build.py --bounds > $O/build.log 2>&1; echo bounds_build=$?
export DTR_LIB=$PWD/paper_2006_09616_b200/libdtr_bounds.so
for c in cta cta_global grid pool_argmin percall adversary; do
  timeout 600 python tools/sanitize_cases.py $c > $O/bounds_$c.log 2>&1; echo "bounds $c rc=$? $(tail -1 $O/bounds_$c.log)"
done | tee $O/summary.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_adversary.py -m gpu -x -q \
    > $O/bounds_pytest.log 2>&1; echo "bounds pytest rc=$? $(tail -1 $O/bounds_pytest.log)" | tee -a $O/summary.txt
