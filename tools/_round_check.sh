#!/bin/bash
# Round re-entry check on a GPU box: gpu tests, smoke, default bench line, and the other workloads.
mkdir -p gpurun_out/chk
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/chk/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/chk/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/chk/smoke.log
for W in bert_large_dgc_allgather bert_large_dgc_alltoall resnet50_efsignsgd_alltoall gpt2_medium_mixed; do
  timeout 600 python bench.py --workload $W --steps 30 --warmup 5 > gpurun_out/chk/bench_$W.json 2> gpurun_out/chk/bench_$W.err; echo "bench $W rc=$?"
  cat gpurun_out/chk/bench_$W.json
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/chk/ref.json 2> gpurun_out/chk/ref.err; echo "ref rc=$?"; cat gpurun_out/chk/ref.json
