lib=paper_2605_18404_b200/libjanus_b200.so
cp $lib /tmp/def.so
for v in c3old c3new c3old c3new; do cp build/var_$v/libjanus_b200.so $lib; r=$(timeout 300 python tools/c3_report.py --nmb 16 --Ps 1 --methods symfold --out /tmp/x.json 2>/dev/null | head -1); echo "$v $r" >> gpurun_out/c3ab.txt; done
cp /tmp/def.so $lib
