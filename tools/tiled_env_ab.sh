# A/B of runtime env settings of the tiled decode kernels (one build):
#   bash tools/tiled_env_ab.sh "LRC_TILED_DYN=0" "LRC_TILED_DYN=1" ...
# -> gpurun_out/te.log (bench B=1/2/4 tokens/s and phase times, B=1 stamps per setting; each setting twice)
for rep in 1 2; do
for v in "$@"; do
  echo "== $v (rep $rep)" >> gpurun_out/te.log
  for b in 1 2 4; do
    env $v timeout 300 python bench.py --batch $b --steps 1000 --warmup 10 --no-sweep --no-prefill --no-offload --no-int3 \
      --no-c5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$b', round(d['value']), d['roofline']['phase_ms'])" >> gpurun_out/te.log
  done
  [ $rep = 1 ] && env $v timeout 100 python tools/route_stamps.py 1 2>&1 | grep -E "^  (up|down) (cons|epi)" >> gpurun_out/te.log
done
done
