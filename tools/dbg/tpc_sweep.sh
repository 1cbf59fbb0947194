# tiles-per-CTA sweep of the TC edge kernels (JANUS_TPC_FE / JANUS_TPC_WG), bench value + e2e
for cfg in "2 4" "2 6" "2 8" "3 4" "3 6" "4 4" "4 8" "4 16" "8 8"; do
  set -- $cfg
  v=$(JANUS_TPC_FE=$1 JANUS_TPC_WG=$2 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e_host_csr']['value'],1))")
  echo "fe=$1 wg=$2 $v"
done
