# attribution: step time with kernel families dropped (JANUS_PROF_SKIP, numerically invalid runs)
for m in 0 1 2 4 8 15 31 63 127 255; do
  v=$(JANUS_PROF_SKIP=$m timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3))")
  echo "skip=$m ms_per_step=$v"
done
