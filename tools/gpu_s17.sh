# the 180 MSPS cells of config 5, each to its end (long)
set -x
O=gpurun_out/r02e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2900 python tools/msps_sweep.py > $O/msps_sweep.json 2>&1; echo msps=$?; cat $O/msps_sweep.json
