# A/B of compile-time variants of the tcd kernel on one box:
#   bash tools/build_variants.sh "-DTCD_WAIT=0" "-DTCD_WAIT=1 -DTCD_ONE_NAS=2" ...
# -> gpurun_out/wv.log (layer step time at B=1 per variant, parity lines)
for v in "$@"; do
  LRC_NVCC_EXTRA="$v" python -m paper_2512_17073_b200.build --force > gpurun_out/bv.log 2>&1 || { echo "build failed: $v" >> gpurun_out/wv.log; continue; }
  echo "== $v" >> gpurun_out/wv.log
  LRC_TCD_MAX=8 timeout 100 python tools/tcd_stamps.py 1 2>&1 | grep -E "5 end|U fin|plan " >> gpurun_out/wv.log
  LRC_TCD_MAX=8 timeout 300 python tools/tcd_check.py --quick 2>&1 | grep -E "timing|B=1: rel" >> gpurun_out/wv.log
done
