for cfg in "256 4 0.3" "0 4 0.3" "0 2 0.3" "0 3 0.3" "0 4 0.6" "0 4 1.0"; do set -- $cfg
  v=$(JANUS_TC_TILE_EDGES=$1 JANUS_TC_TILE_MAXCH=$2 JANUS_TC_TILE_OVH=$3 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), round(d['value'],1), round(d['e2e']['value'],1))")
  c5=$(JANUS_TC_TILE_EDGES=$1 JANUS_TC_TILE_MAXCH=$2 JANUS_TC_TILE_OVH=$3 timeout 300 python tools/config_bench.py 2>/dev/null | grep C5 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['structures_per_s'],1))")
  echo "te=$1 maxch=$2 ovh=$3 C2: $v  C5: $c5"
done
