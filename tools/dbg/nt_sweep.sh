# 512- vs 1024-thread tensor-core edge kernels: tf32 parity tests + bench
JANUS_LIB=build/nt1024/libjanus_b200.so timeout 600 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_c5.py tests/test_gpu_tc.py -x -q 2>&1 | tail -3
for lib in paper_2605_18404_b200/libjanus_b200.so build/nt1024/libjanus_b200.so; do
  for cfg in "4 8" "2 4" "1 2"; do set -- $cfg
  v=$(JANUS_LIB=$lib JANUS_TPC_FE=$1 JANUS_TPC_WG=$2 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3), round(d['value'],1), round(d['roofline']['launch_ms']*1000,2))")
  echo "$lib tpc=$1/$2 $v"
  done
done
