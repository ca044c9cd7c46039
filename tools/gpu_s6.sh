# session 4c: stream scoring for global-state CTA cells, pipelined closure pass, full-length parity
set -x
mkdir -p gpurun_out/s6
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s6/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fulllength" > gpurun_out/s6/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s6/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_fulllength.py -x -q -s > gpurun_out/s6/pytest_full.log 2>&1; echo pytest_full=$?; tail -5 gpurun_out/s6/pytest_full.log
python paper_2006_09616_b200/_build.py --profile > /dev/null 2>&1; echo profbuild=$?
for c in "transformer msps 317 3000" "densenet100 msps 317 3000" "lstm msps 317 3000" "lstm dtr_eq 317 20000" "lstm dtr 100 20000" "treelstm dtr 100 20000"; do
  timeout 300 python tools/probe_prof_c5.py $c 2>&1 | tail -4
done > gpurun_out/s6/prof.log; cat gpurun_out/s6/prof.log
for m in transformer treelstm lstm; do
  OUT=gpurun_out/s6/c5_groups.jsonl timeout 300 python tools/probe_c5_groups.py dtr,dtr_eq $m 2>&1 | tail -2
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cta_engine -s 1 -c 1 -o gpurun_out/s6/cta_lstm \
    python tools/one_cell_c5.py lstm dtr 100 5000 2 > gpurun_out/s6/ncu_lstm.log 2>&1; echo ncu=$?
ncu -i gpurun_out/s6/cta_lstm.ncu-rep --page raw --csv > gpurun_out/s6/cta_lstm_raw.csv 2>/dev/null
ncu -i gpurun_out/s6/cta_lstm.ncu-rep --page details --csv > gpurun_out/s6/cta_lstm_details.csv 2>/dev/null
rm -f gpurun_out/s6/cta_lstm.ncu-rep
