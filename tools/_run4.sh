python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --no-cpu-baseline --steps 50 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', round(d['value']), round(d['ms_per_step'],4))"
python bench.py --no-cpu-baseline --workload gpt2_medium_mixed --steps 30 --warmup 5 --phases 2>gpurun_out/g.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpt2 N=1', round(d['value']), round(d['ms_per_step'],4))"
grep phases gpurun_out/g.err
python tools/dbg_big.py dgc 0.01 28; python tools/dbg_big.py dgc 0.001 28; python tools/dbg_big.py topk 0.001 28
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/big.csv python tools/dbg_big.py dgc 0.01 28 >/dev/null 2>&1; python tools/launches.py gpurun_out/big.csv 9
