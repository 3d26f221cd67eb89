#!/bin/bash
# A/B of bench.py argument sets on one workload at N=1: bash tools/_ab_args.sh WORKLOAD "ARGS1" "ARGS2" ...
W=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do for A in "$@"; do
  [ "$A" = "-" ] && AA="" || AA="$A"
  timeout 300 python bench.py --workload $W --steps 100 --warmup 10 --e2e-steps 0 --no-cpu-baseline $AA > /tmp/o.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print(f'{\"$A\":30s} mean {d[\"ms_per_step\"]:.4f} med {d[\"config\"][\"median_ms_per_step\"]:.4f}')"
done; done
