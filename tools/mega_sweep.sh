#!/bin/bash
# far-field planner sweep at cfg2 (tuning aid): work-area budget x bottom split level x near ring depth
for b in 5800 7000 8200 9400; do for ls in 0 6 7 8; do
  echo "budget $b ls>=$ls: $(H2B_MEGA_BUDGET=$b H2B_DEBUG_LS=$ls python tools/quick_time.py 2 2>&1 | tail -1)"
done; done
for n in 4 5 6 7; do echo "nst $n: $(H2B_DEBUG_NEAR_NST=$n python tools/quick_time.py 2 2>&1 | tail -1)"; done
