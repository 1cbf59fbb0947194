# Chunks-per-CTA sweep of the pair (JANUS_TPC_WG) and filter (JANUS_TPC_FE)
# kernels on the C2 workload (tools/config_bench.py; the knobs are tuning
# switches, which bench.py refuses).  Usage: bash tools/sweep_tpc.sh [out]
out=${1:-gpurun_out/sweep.txt}; rm -f $out
run () { r=$(env $1 timeout 200 python tools/config_bench.py --only C2 2>/dev/null | tail -1); echo "$1 $r" | cut -c1-160 >> $out; }
for rep in 1 2; do
  for wg in 5 7 10; do run "JANUS_TPC_WG=$wg"; done
  for fe in 2 5; do run "JANUS_TPC_FE=$fe"; done
done
