for b in 16 32 64; do
  for v in "X=1" "LRC_PREFILL_MIN=9"; do
    env $v timeout 300 python bench.py --batch $b --steps 200 --warmup 5 --no-sweep --no-prefill --no-offload --no-int3 --no-c5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$b $v', round(d['value']), d['roofline']['phase_ms'])" >> gpurun_out/pf.log
  done
done
