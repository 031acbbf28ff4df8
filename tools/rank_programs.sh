#!/bin/bash
# per-rank device programs of the subtree partition (tools/rank_programs.py): cfg3 with parity
# against the single-GPU operator at G = 8, then the 2M-unknown cube (cfg4) at G = 2, 4, 8
python tools/rank_programs.py fixtures/cfg3_structure.npz 8 --check
for G in 1 2 4; do python tools/rank_programs.py fixtures/cfg3_structure.npz $G | tail -1; done
for G in 8 4 2; do python tools/rank_programs.py fixtures/cfg4_structure.npz $G; done
