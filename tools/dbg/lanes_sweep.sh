for cfg in "16 2 3" "24 2 3" "32 2 3" "32 1 2" "32 2 4" "12 2 3"; do set -- $cfg
  v=$(JANUS_TPC_FE=$2 JANUS_TPC_WG=$3 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --lanes $1 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), round(d['value'],1), round(d['e2e']['value'],1))")
  echo "lanes=$1 tpc=$2/$3 $v"
done
