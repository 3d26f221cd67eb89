#!/bin/bash
# NCCL-world parity at 1..G processes + scaling bench of the fused paths (run via gpurun --gpus G)
G=${1:-2}
mkdir -p gpurun_out/nccl
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py -x -q > gpurun_out/nccl/pytest.log 2>&1; echo "nccl pytest rc=$?"; tail -30 gpurun_out/nccl/pytest.log
