python -m pytest tests -m gpu -x -q -k "dgc or topk or config1 or pairs" 2>&1 | tail -1
for V in 0 4; do for S in 4 6; do
  ESP_TMA_VARIANT=$V ESP_TMA_STAGES=$S python bench.py --no-cpu-baseline --phases --steps 50 --warmup 5 2>gpurun_out/ph.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('V=$V S=$S bench', round(d['ms_per_step'],4), d['roofline']['achieved'], end=' ')"
  grep -i phase gpurun_out/ph.err | tail -1 | python -c "import sys,json; s=sys.stdin.read(); d=json.loads(s[s.index('{'):]); print('h1', round(d['h1_ms'],4))"
done; done
