mkdir -p gpurun_out
TAG=${1:-kexp}; W=${2:-r50_stem}
timeout 900 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --warp-sampling-max-passes 20 --import-source on --clock-control none -k regex:k_explore_gens -s 2 -c 1 -o /tmp/$TAG -f python tools/probe_explore.py $W > gpurun_out/ncu_$TAG.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>>gpurun_out/ncu_$TAG.log
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_source.csv 2>>gpurun_out/ncu_$TAG.log
