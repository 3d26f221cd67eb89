set -e
python -m pytest tests -m gpu -x -q -k "parity" 2>&1 | tail -2
python bench.py --no-cpu-baseline --phases --steps 50 --warmup 5 2>gpurun_out/ph.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['frac'])"
grep -i phase gpurun_out/ph.err | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches8.csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 0 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches8.csv 5 | grep h2
