#!/bin/bash
# Profiling pass of one round on a GPU box (run via gpurun; results in gpurun_out/prof/).
#   1. the plain bench line (no profiler)
#   2. the launch list of the same command (ncu, gpu__time_duration.sum, clocks not locked)
#   3. one `ncu --set full` capture of every kernel of one steady-state step
set -e
W=${1:-bert_large_dgc_allgather}
mkdir -p gpurun_out/prof
[ -n "$NOBENCH" ] || python bench.py --workload $W --steps 50 --warmup 5 > gpurun_out/prof/bench_$W.json 2> gpurun_out/prof/bench_$W.err
cat gpurun_out/prof/bench_$W.json 2>/dev/null || true
[ -n "$NOBENCH" ] || ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$W.csv \
  python bench.py --workload $W --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
[ -n "$NOBENCH" ] || python tools/launches.py gpurun_out/prof/launches_$W.csv 5 > gpurun_out/prof/launches_$W.txt
cat gpurun_out/prof/launches_$W.txt 2>/dev/null || true
ncu --set full --clock-control none --import-source on -k regex:"dgc_|h2_" --launch-skip ${SKIP:-24} -c ${COUNT:-8} \
  -o gpurun_out/prof/full_$W python bench.py --workload $W --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
  > gpurun_out/prof/full_$W.log 2>&1
tail -2 gpurun_out/prof/full_$W.log
