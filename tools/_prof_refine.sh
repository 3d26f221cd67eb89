#!/bin/bash
# ncu --set full of the DGC finalize chain (refine x2, write) of one steady-state BERT-large step.
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dgc_refine|dgc_write|dgc_sample" --launch-skip 12 -c 4 \
  -o gpurun_out/prof/finalize_bert python bench.py --workload bert_large_dgc_allgather --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > gpurun_out/prof/finalize_bert.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/prof/finalize_bert.log
