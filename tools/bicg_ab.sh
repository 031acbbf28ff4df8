#!/bin/bash
# BiCGStab at cfg1: graph-driven loop with fused cluster segments / unfused segments / host loop
for v in fused unfused host fused; do
  unset H2B_BICG_HOST H2B_BICG_UNFUSED
  if [ $v = host ]; then export H2B_BICG_HOST=1; fi
  if [ $v = unfused ]; then export H2B_BICG_UNFUSED=1; fi
  echo "$v: $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d["bicgstab"]))')"
done
