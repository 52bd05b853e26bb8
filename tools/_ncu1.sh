mkdir -p gpurun_out
KRE=${1:-k_fsel}; TAG=${2:-kfsel}; shift 2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$KRE" -s 2 -c 1 -o /tmp/$TAG -f python tools/one_round.py "$@" > gpurun_out/ncu_$TAG.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>>gpurun_out/ncu_$TAG.log
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>>gpurun_out/ncu_$TAG.log
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_source.csv 2>>gpurun_out/ncu_$TAG.log
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_cuda.csv 2>>gpurun_out/ncu_$TAG.log
[ -n "$KEEP_REP" ] && cp /tmp/$TAG.ncu-rep gpurun_out/ 2>/dev/null
rm -f gpurun_out/${TAG}_cuda.csv  # large; the SASS page carries the stalls
