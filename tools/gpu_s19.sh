set -x
O=gpurun_out/r02g
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_fulllength.py -x -q -s > $O/pytest_full.log 2>&1; echo full=$?; tail -5 $O/pytest_full.log
