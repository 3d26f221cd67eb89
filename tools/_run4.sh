python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for G in x 1 3; do
if [ $G = x ]; then unset ESP_TMA_GROUPS; else export ESP_TMA_GROUPS=$G; fi
python bench.py --no-cpu-baseline --workload gpt2_medium_mixed --steps 30 --warmup 5 --phases 2>gpurun_out/g.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G=$G gpt2 N=1', round(d['value']), round(d['ms_per_step'],4), end=' ')"
grep phases gpurun_out/g.err | python -c "import sys,json; s=sys.stdin.read(); d=json.loads(s[s.index('{'):]); print('h1', round(d['h1_ms'],4), 'mid', round(d['mid_ms'],4), 'h2', round(d['h2_ms'],4))"
python bench.py --no-cpu-baseline --workload resnet50_efsignsgd_alltoall --steps 50 --warmup 5 --phases 2>gpurun_out/r.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G=$G resnet N=1', round(d['value']), round(d['ms_per_step'],4), end=' ')"
grep phases gpurun_out/r.err | python -c "import sys,json; s=sys.stdin.read(); d=json.loads(s[s.index('{'):]); print('h1', round(d['h1_ms'],4), 'mid', round(d['mid_ms'],4), 'h2', round(d['h2_ms'],4))"
done
