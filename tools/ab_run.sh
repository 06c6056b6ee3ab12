# A/B of libvdc builds on one box: abtest/libvdc_<name>.so for each name in $AB (C2 rounds, then C3)
set -x
AB=${AB:-"w12mma fold"}
for r in $(seq 1 ${AB_C2_ROUNDS:-3}); do
for v in $AB; do
  VDC_LIB=abtest/libvdc_$v.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/ab2_c2_${v}_$r.json 2>gpurun_out/ab2_err_$v.txt
done
done
for r in $(seq 1 ${AB_C3_ROUNDS:-0}); do
for v in $AB; do
  VDC_LIB=abtest/libvdc_$v.so timeout 300 python bench.py --batch 32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab2_c3_${v}_$r.json 2>>gpurun_out/ab2_err_$v.txt
done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab2_c*.json")):
    try:
        d=json.load(open(f)); print(f, d["value"], d["roofline"]["frac"], d["e2e"]["value"])
    except Exception as e: print(f, "ERR", e)
PY
