#!/bin/bash
# tuning aid: near-field start delay vs step time at cfg2
for d in 0 2000 4000 6000 8000 10000 0; do echo "delay $d ns: $(H2B_DEBUG_NEAR_DELAY_NS=$d python tools/quick_time.py 2 2>&1 | tail -1)"; done
