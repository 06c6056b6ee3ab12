# End-of-round measurements on one B200 (outputs under gpurun_out/final/):
# GPU tests, the bench lines (C2 default, resident, C3, C4 on one GPU, the
# reference arm), the ncu launch list and one --set full capture per kernel.
set -x
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.txt 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --resident 20 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2_resident20.json 2> $O/bench_res.err
timeout 600 python bench.py --batch 32 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_batch32.json 2> $O/bench_c3.err
timeout 600 python bench.py --batch 8 --model qwen3-8b --ctx-fixed 4096 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4_qwen3_batch8_1gpu.json 2> $O/bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference_arm.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_kernel -s 3 -c 1 -f -o $O/prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ring_kernel -s 3 -c 1 -f -o $O/prof_c3 python bench.py --batch 32 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c3.log 2>&1
tail -1 $O/gpu_tests.txt
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d.get('value'), d.get('roofline',{}).get('frac'), d.get('e2e',{}).get('value'))"; done
ls -la $O
