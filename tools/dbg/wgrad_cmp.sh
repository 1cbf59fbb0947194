for e in 0 1 0 1; do
  if [ $e = 1 ]; then export JANUS_WGRAD_SIMT=1; else unset JANUS_WGRAD_SIMT; fi
  v=$(timeout 100 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), round(d['value'],1))")
  echo "simt=$e $v"
done
