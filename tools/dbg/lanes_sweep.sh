for l in 8 16 24 32; do
  v=$(timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --lanes $l 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), round(d['value'],1))")
  v2=$(JANUS_PROF_SKIP=15 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --lanes $l 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3))")
  echo "lanes=$l $v  no-edge: $v2"
done
