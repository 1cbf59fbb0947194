for cfg in "1 3 32" "2 3 32" "1 4 32" "1 3 16" "2 3 16"; do set -- $cfg
  v=$(JANUS_TPC_FE=$1 JANUS_TPC_WG=$2 timeout 100 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --lanes $3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), round(d['value'],1))")
  echo "tpc=$1/$2 lanes=$3 $v"
done
