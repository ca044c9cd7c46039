# ncu --set full of dtr_pool_argmin at the 1e6 pool (+ source page)
set -x
O=gpurun_out/${1:-pa}
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_argmin -s 2 -c 1 -o $O/pa_full \
    python scripts/pool_argmin_one.py 1000000 ${2:-0} > $O/ncu_pa.log 2>&1; echo ncu_pa=$?
ncu -i $O/pa_full.ncu-rep --page raw --csv > $O/pa_raw.csv 2>/dev/null
ncu -i $O/pa_full.ncu-rep --page details --csv > $O/pa_details.csv 2>/dev/null
ncu -i $O/pa_full.ncu-rep --page source --csv --print-source sass > $O/pa_source_sass.csv 2>/dev/null
ncu -i $O/pa_full.ncu-rep --page source --csv --print-source cuda > $O/pa_source_cuda.csv 2>/dev/null
ls -la $O
