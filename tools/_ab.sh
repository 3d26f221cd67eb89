#!/bin/bash
# A/B of env knobs on one workload at N ranks (run via gpurun --gpus N):
#   bash tools/_ab.sh N WORKLOAD "ENV1" "ENV2" ...   (each ENV a space-separated list of VAR=VAL, or "-")
N=$1; W=$2; shift 2
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for E in "$@"; do
  [ "$E" = "-" ] && EE="" || EE="$E"
  if [ $N = 1 ]; then L="python"; else L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513"; fi
  env $EE timeout 300 $L bench.py --gpus $N --workload $W --steps 100 --warmup 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab/o.json 2> gpurun_out/ab/o.err
  python - "$E" <<'PY'
import json,sys
try:
  d=json.loads(open("gpurun_out/ab/o.json").read().strip().splitlines()[-1]); r=d['roofline']
  print(f"{sys.argv[1]:40s} mean {d['ms_per_step']:.4f} med {d['config']['median_ms_per_step']:.4f} kern {r['kernel_ms_per_step']:.4f}")
except Exception as ex: print(sys.argv[1],'FAIL',ex, open("gpurun_out/ab/o.err").read()[-800:])
PY
done; done
