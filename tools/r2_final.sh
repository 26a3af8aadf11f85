# Final round-2 evidence run (one GPU): GPU test suite, full bench, ncu launch
# list of the decode bench command, one ncu --set full capture of tiled_kernel UP.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_gputests.txt 2>&1
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"route_kernel|tiled_kernel|lr_down_kernel|tcd_kernel|prefill_kernel|gate" -c 300 --csv \
  --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 100 --warmup 5 --no-sweep --no-cpu-baseline --no-prefill --no-offload --no-int3 --no-c5 \
  > gpurun_out/final_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tiled_kernel -s 40 -c 2 \
  -o gpurun_out/final_tiled python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --no-prefill \
  --no-offload --no-int3 --no-c5 > gpurun_out/final_ncu_tiled.log 2>&1
