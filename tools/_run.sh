set -e
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline --phases --steps 50 --warmup 5 2>gpurun_out/ph.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['frac'])"
grep -i phase gpurun_out/ph.err | tail -1
for w in bert_large_dgc_alltoall resnet50_efsignsgd_alltoall gpt2_medium_mixed; do python bench.py --no-cpu-baseline --workload $w --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'])"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7.csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 0 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches7.csv 5
