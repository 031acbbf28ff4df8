#!/bin/bash
# GMRES(30) at cfg1: fused single-cluster Arnoldi step vs the multi-kernel step (A/B)
for v in fused multi fused multi; do
  if [ $v = multi ]; then export H2B_NO_FUSED_ARNOLDI=1; else unset H2B_NO_FUSED_ARNOLDI; fi
  echo "$v: $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d["gmres"]))')"
done
