# Round evidence, part B: compute-sanitizer over every kernel, the MSPS cells of the
# config-5 sweep, the App. A residency trace.  usage: bash tools/gpu_evidence_b.sh TAG
set -x
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/residency_trace.py 200 $O/residency_N200_estar_v1 > $O/residency.log 2>&1; echo resid=$?; cat $O/residency.log
bash tools/sanitize.sh $O/sanitize
timeout 2400 python tools/msps_sweep.py > $O/msps_sweep.json 2>&1; echo msps=$?; cat $O/msps_sweep.json
