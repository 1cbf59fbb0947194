out=gpurun_out/sweep.txt; rm -f $out
for wg in 3 4 5 7; do for rep in 1 2; do r=$(JANUS_TPC_WG=$wg timeout 200 python tools/config_bench.py --only C2 2>/dev/null | tail -1); echo "wg=$wg $r" | cut -c1-120 >> $out; done; done
