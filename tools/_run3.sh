python -m pytest tests -m gpu -x -q -k "dgc or topk" 2>&1 | tail -1
ESP_TMA_STAGES=6 python -m pytest tests -m gpu -x -q -k "dgc" 2>&1 | tail -1
for VS in "0 4" "0 6" "8 4" "8 6" "0 4"; do set -- $VS
  ESP_TMA_VARIANT=$1 ESP_TMA_STAGES=$2 python bench.py --no-cpu-baseline --phases --steps 50 --warmup 5 2>gpurun_out/ph_$1_$2.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('V=$1 S=$2 bench', round(d['ms_per_step'],4), round(d['roofline']['achieved']))"
done
