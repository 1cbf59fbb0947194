#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   bench line, ncu launch list of one bench step, ncu --set full of the
#   largest edge kernel (msg_bf_pair_tc) and the node weight-gradient kernel
#   (wgrad_tc_kernel), phase traces of the TC edge kernels.
# Outputs land in gpurun_out/<tag>_*; copy the summaries into profiles/.
set -u
tag=${1:-prof}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py --steps 20 --warmup 5 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1
gzip -f $out/${tag}_launches.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:msg_bf_pair_tc -s 40 -c 1 \
  -o $out/${tag}_msg_bf_pair_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_tc_kernel -s 200 -c 1 \
  -o $out/${tag}_wgrad_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_full_wg.log 2>&1
if [ -f build/trace/libjanus_b200.so ]; then
  JANUS_LIB=build/trace/libjanus_b200.so timeout 200 python tools/tc_trace.py > $out/${tag}_trace.txt 2>&1
fi
ls -la $out | grep $tag
# device LM (nbrlist.cu): full capture of the fill kernel on the batched C2 x 32 build
timeout 300 ncu --set full --clock-control none -k regex:fill_kernel -s 280 -c 1 \
  -o $out/${tag}_nbr_fill python tools/nbrlist_bench.py > $out/${tag}_ncu_nbr.log 2>&1
