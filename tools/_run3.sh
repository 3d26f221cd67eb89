for T in 1024 2048 4096 1024 512; do
  ESP_NVCC_EXTRA="-DESP_H2_TILE=$T" python paper_2205_14465_b200/build.py --force > /dev/null
  for rep in 1 2; do
  python bench.py --no-cpu-baseline --phases --steps 50 --warmup 5 2>gpurun_out/ph.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('T=$T bench', round(d['ms_per_step'],4), end=' ')"
  grep -i phase gpurun_out/ph.err | tail -1 | python -c "import sys,json; s=sys.stdin.read(); d=json.loads(s[s.index('{'):]); print('h2', round(d['h2_ms'],4))"
  done
done
