python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for N in 2 4; do
for w in bert_large_dgc_allgather gpt2_medium_mixed; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --workload $w --no-cpu-baseline --steps 30 --warmup 5 --phases 2>gpurun_out/mg_${N}_$w.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N $w', round(d['value']), round(d['ms_per_step'],4))"
grep -h "phases" gpurun_out/mg_${N}_$w.err | tail -1
done; done
