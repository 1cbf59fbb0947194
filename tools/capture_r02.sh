#!/bin/bash
# Round-2 profile capture (run on the GPU box from the repo root):
#   bench line; ncu launch list of one bench step; ncu --set full of the
#   hot kernels (pair, filter, row, upd and neighbour-list kernels).
# Outputs land in gpurun_out/<tag>_*; tools/ncu_summary.py turns the .ncu-rep
# files into the summaries kept under profiles/.
set -u
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py --steps 30 --warmup 5 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fp32-path > $out/${tag}_ncu_launch.log 2>&1
gzip -f $out/${tag}_launches.csv
for k in msg_bf_pair_tc msg_be_pair_tc msg_filter_tc msg_fe_rows msg_ff_rows msg_bf_rows msg_be_rows upd_bf_tc upd_fe_tc wgrad_tc_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 40 -c 1 \
    -o $out/${tag}_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp32-path > $out/${tag}_ncu_$k.log 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:"walk_pad" -c 1 -o $out/${tag}_walk_pad python tools/e2e_probe.py --steps 1 > $out/${tag}_ncu_walk.log 2>&1
ls -la $out | grep $tag
# summaries on the box; keep only the top kernel's report (gpurun returns <= 64 MiB)
python tools/ncu_summary.py $out/${tag}_*.ncu-rep > $out/${tag}_ncu_summary.json 2> $out/${tag}_ncu_summary.err
for f in $out/${tag}_*.ncu-rep; do
  case $f in *msg_bf_pair_tc*) ;; *) rm -f $f ;; esac
done
