#!/bin/bash
# A/B two liblrc.so builds (var_<a>.so, var_<b>.so), keep the faster at B=1
# (B=8 not more than 2% worse), then parity tests + smoke + full bench on it.
L=paper_2512_17073_b200/_lib
A=$1; B=$2
bash tools/unroll_sweep.sh $A $B $A $B > gpurun_out/ab.log 2>&1
W=$(python - "$A" "$B" <<'PY'
import re, sys
a, b = sys.argv[1:3]
v = {}
for line in open("gpurun_out/ab.log"):
    m = re.match(r"(\S+) B=(\d+) -> ([\d.]+)", line)
    if m: v.setdefault((m[1], m[2]), []).append(float(m[3]))
mean = lambda k: sum(v[k]) / len(v[k])
ok = mean((b, "1")) > mean((a, "1")) and mean((b, "8")) > 0.98 * mean((a, "8"))
print(b if ok else a)
PY
)
echo "winner=$W" | tee gpurun_out/winner.txt
cp $L/var_$W.so $L/liblrc.so
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/parity_w.log 2>&1; echo parity_rc=$? | tee -a gpurun_out/winner.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_w.log 2>&1; echo smoke_rc=$? | tee -a gpurun_out/winner.txt
python bench.py > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err; echo bench_rc=$? | tee -a gpurun_out/winner.txt
