#!/bin/bash
# A/B of library builds on the GPU box: for each build/var_*/libjanus_b200.so,
# install it in-tree and run the bench (device value, e2e, roofline), then
# restore the default build.  Usage: bash tools/ab_libs.sh <out> [steps] var1 var2 ...
out=$1; steps=$2; shift 2
lib=paper_2605_18404_b200/libjanus_b200.so
cp $lib /tmp/janus_default.so
for rep in 1 2; do
  for v in "$@"; do
    cp build/var_$v/libjanus_b200.so $lib
    r=$(timeout 300 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-fp32-path 2>/dev/null | tail -1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print(sys.argv[2], sys.argv[3], round(d['value']), round(d['e2e']['value']), round(d['roofline'].get('achieved',0),1))" "$r" "$v" "$rep" >> $out
  done
done
cp /tmp/janus_default.so $lib
