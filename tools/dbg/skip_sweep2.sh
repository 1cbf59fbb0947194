for m in 0 64 128 15 79 143 255; do
  v=$(JANUS_PROF_SKIP=$m timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --lanes 32 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3))")
  echo "lanes32 skip=$m ms_per_step=$v"
done
