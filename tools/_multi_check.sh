#!/bin/bash
# Multi-GPU re-entry check (run via gpurun --gpus G): full gpu suite incl. the multi-rank cases, then the scaling table.
G=${1:-4}
mkdir -p gpurun_out/multi
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/multi/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -8 gpurun_out/multi/pytest_gpu.log
bash tools/_scale.sh $G | tee gpurun_out/multi/scaling.txt
