# Round-2 evidence run (one GPU): full bench, ncu launch list of the decode
# bench command, one ncu --set full capture of the dominant decode kernel
# (tiled_kernel UP) and of the tensor-core decode engine (INT3 C2, B=1).
set -x
timeout 1200 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"route_kernel|tiled_kernel|lr_down_kernel|tcd_kernel|prefill_kernel|gate" -c 300 --csv \
  --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu-baseline --no-prefill --no-offload --no-int3 \
  > gpurun_out/r2_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tiled_kernel -s 40 -c 1 \
  -o gpurun_out/r2_tiled_up python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-prefill \
  --no-offload --no-int3 > gpurun_out/r2_ncu_tiled.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tcd_kernel -s 6 -c 1 \
  -o gpurun_out/r2_tcd_int3 python tools/gen3_profile.py 1 tcd > gpurun_out/r2_ncu_tcd.log 2>&1
