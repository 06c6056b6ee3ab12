for cfg in "128 -1" "256 -1" "96 -1" "128 16" "128 30" "192 -1"; do
  set -- $cfg
  v=$(timeout 300 python bench.py --batch 32 --steps 10 --warmup 3 --no-cpu-baseline --pages-per-job $1 --attn-job-cost $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])" 2>&1 | tail -1)
  echo "ppj $1 cost $2: $v"
done
