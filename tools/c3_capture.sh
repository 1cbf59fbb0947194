#!/bin/bash
# configs[2] evidence on the GPU box: the C3 report (P = 1 and 8), a launch
# list of a short C3 run (L = 4, one lane) and one ncu --set full capture of
# each fused-epilogue GEMM (gemm_tc.cuh).  Usage: bash tools/c3_capture.sh TAG
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 python tools/c3_report.py --out gpurun_out/${tag}_c3_report.json > gpurun_out/${tag}_c3_report.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c3_launches.csv \
  python tools/c3_report.py --nmb 2 --L 4 --Ps 1 --methods symfold --lanes 1 --out /tmp/x.json > /dev/null 2>&1
for e in EpiAct2 EpiFilter EpiZbar EpiAct1 EpiBeZbar; do
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:$e -s 2 -c 1 \
    -o gpurun_out/${tag}_gemm_$e python tools/c3_report.py --nmb 2 --L 2 --Ps 1 --methods symfold --lanes 1 --out /tmp/x.json > /dev/null 2>&1
done
