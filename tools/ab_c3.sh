# A/B of library variants on configs[2] (C3): each build/var_<v>/libjanus_b200.so
# in turn, SymFold P=1, results appended to gpurun_out/c3ab.txt.
# Usage: bash tools/ab_c3.sh v1 v2 ...   (interleave the list to cancel drift)
for v in "$@"; do
  r=$(JANUS_LIB=build/var_$v/libjanus_b200.so timeout 300 python tools/c3_report.py --nmb 16 --Ps 1 --methods symfold --out /tmp/x.json 2>/dev/null | head -1)
  echo "$v $r" >> gpurun_out/c3ab.txt
done
