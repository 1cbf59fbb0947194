#!/bin/bash
# Step attribution on the GPU box: C2 step time with kernel classes skipped
# (make PROFILE=1 build, JANUS_PROF_SKIP bit mask: 1 FE edge, 2 FF edge,
# 4 BF edge, 8 BE edge, 16 node weight gradients, 32 upd units, 64 row GEMMs,
# 128 partial reductions).  Never a bench line: the profiling build drops work.
out=$1
for m in 0 16 32 64 4 8 12 1 2 255; do
  r=$(JANUS_LIB=build/prof/libjanus_b200.so JANUS_PROF_SKIP=$m timeout 300 python tools/config_bench.py --only C2 2>/dev/null | tail -1)
  echo "skip=$m $r" >> $out
done
