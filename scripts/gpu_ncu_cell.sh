# ncu --set full (+ source) of one config-2 cell on the CTA engine: bash scripts/gpu_ncu_cell.sh TAG H PERMILLE
set -x
O=gpurun_out/${1:-cell}
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cta_engine -s 1 -c 1 -o $O/cell \
    python scripts/one_cell.py ${2:-3} ${3:-100} 2 > $O/ncu_cell.log 2>&1; echo ncu=$?
ncu -i $O/cell.ncu-rep --page raw --csv > $O/cell_raw.csv 2>/dev/null
ncu -i $O/cell.ncu-rep --page details --csv > $O/cell_details.csv 2>/dev/null
ncu -i $O/cell.ncu-rep --page source --csv --print-source sass > $O/cell_source_sass.csv 2>/dev/null
rm -f $O/cell.ncu-rep
