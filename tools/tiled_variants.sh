# A/B of compile-time variants of the tiled decode kernels on one box:
#   bash tools/tiled_variants.sh "" "-DTILED_NW1=16 -DTILED_SPAN1=2" ...
# -> gpurun_out/tv.log (bench B=1/2/4 tokens/s and phase times, B=1 stamps per variant)
for v in "$@"; do
  LRC_NVCC_EXTRA="$v" python -m paper_2512_17073_b200.build --force > gpurun_out/bv.log 2>&1 || { echo "build failed: $v" >> gpurun_out/tv.log; continue; }
  echo "== $v" >> gpurun_out/tv.log
  for b in 1 2 4; do
    timeout 300 python bench.py --batch $b --steps 1000 --warmup 10 --no-sweep --no-prefill --no-offload --no-int3 \
      --no-c5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$b', round(d['value']), d['roofline']['phase_ms'])" >> gpurun_out/tv.log
  done
  timeout 100 python tools/route_stamps.py 1 2>&1 | grep -E "^  (up|down) (cons|epi)" >> gpurun_out/tv.log
done
