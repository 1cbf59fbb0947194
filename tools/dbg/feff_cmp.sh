for lib in paper_2605_18404_b200/libjanus_b200.so build/feff1/libjanus_b200.so; do
  echo "== $lib"
  JANUS_LIB=$lib timeout 600 python tools/pipeline_report.py --Ps 4 --out gpurun_out/feff_tmp.json 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print(d['P'], d['method'], d['k'], round(d['structures_per_s'],1))
    except Exception: pass"
  JANUS_LIB=$lib timeout 100 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench', round(d['value'],1))"
done
