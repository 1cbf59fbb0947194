# ncu --set full of each tensor-core edge kernel inside the bench step, then the per-kernel roofline table
out=gpurun_out
for k in msg_fe_tc msg_ff_tc msg_bf_tc msg_be_tc; do
  timeout 400 ncu --set full --clock-control none -k regex:$k -s 40 -c 1 -o $out/v12_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/v12_ncu_$k.log 2>&1
  ncu -i $out/v12_$k.ncu-rep --page raw --csv > $out/v12_$k.csv 2>/dev/null
done
timeout 300 python tools/kernel_roofline.py --ncu-csv msg_fe_tc=$out/v12_msg_fe_tc.csv msg_ff_tc=$out/v12_msg_ff_tc.csv msg_bf_tc=$out/v12_msg_bf_tc.csv msg_be_tc=$out/v12_msg_be_tc.csv --out $out/kernel_roofline.json
