lib=paper_2605_18404_b200/libjanus_b200.so
# A/B of library builds on every config of tools/config_bench.py (GPU box)
cp $lib /tmp/def.so
for v in simtupd updtc simtupd updtc; do cp build/var_$v/libjanus_b200.so $lib; echo "== $v" >> gpurun_out/c1ab.txt; timeout 300 python tools/config_bench.py 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['config'][:12], round(d['structures_per_s']))" >> gpurun_out/c1ab.txt; done
cp /tmp/def.so $lib
