for d in 512; do echo "== dbg $d"; LRC_TCD_DEBUG=$d timeout 100 python tools/tcd_stamps.py 1 | grep -E "plan|dec->D|end|stage"; done
