for e in 0 1 0 1; do
  if [ $e = 1 ]; then export JANUS_LM_LOW_PRIORITY=1; else unset JANUS_LM_LOW_PRIORITY; fi
  v=$(timeout 100 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value'],1), round(d['e2e']['value'],1))")
  echo "low=$e $v"
done
