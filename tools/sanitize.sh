# compute-sanitizer over every kernel (run on a GPU box: bash tools/sanitize.sh OUTDIR).
# NOTE: compute-sanitizer is closed on the round-2 GPU pool; tools/bounds_check.sh is the substitute.
O=${1:-gpurun_out/sanitize}
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  for c in cta cta_global grid pool_argmin percall adversary; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c > $O/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' $O/${tool}_$c.log | tail -1)"
  done
done | tee $O/summary.txt
