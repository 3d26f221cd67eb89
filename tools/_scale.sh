#!/bin/bash
# Multi-GPU scaling check (run via gpurun --gpus G): every workload at N=1..G with phases.
G=${1:-4}
mkdir -p gpurun_out/scale
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for W in bert_large_dgc_allgather bert_large_dgc_alltoall resnet50_efsignsgd_alltoall gpt2_medium_mixed; do
for N in 1 2 $G; do
  if [ $N = 1 ]; then L="python"; else L="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"; fi
  timeout 300 $L bench.py --gpus $N --workload $W --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline --phases > gpurun_out/scale/${W}_$N.json 2> gpurun_out/scale/${W}_$N.err
  python - "$W" "$N" <<'PY'
import json,sys
W,N=sys.argv[1:]
try:
  d=json.loads(open(f"gpurun_out/scale/{W}_{N}.json").read().strip().splitlines()[-1])
  e=open(f"gpurun_out/scale/{W}_{N}.err").read()
  ph=[l for l in e.splitlines() if 'phases' in l]
  print(W,N,round(d['value']),round(d['ms_per_step'],4),ph[-1][:200] if ph else '')
except Exception as ex: print(W,N,'FAIL',ex)
PY
done; done
