#!/bin/bash
# BiCGStab at cfg1: graph-driven loop vs the host-driven loop (A/B)
for v in graph host graph host; do
  if [ $v = host ]; then export H2B_BICG_HOST=1; else unset H2B_BICG_HOST; fi
  echo "$v: $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d["bicgstab"]))')"
done
