#!/bin/bash
# full GPU test suite + a short multi-GPU bench set (run via gpurun --gpus G)
G=${1:-4}; shift
mkdir -p gpurun_out/full
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/full/pytest_gpu.log
for W in "$@"; do bash tools/_ab.sh $G $W -; done
