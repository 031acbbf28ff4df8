#!/bin/bash
# far-field probe: split timings, trace + critical chain at cfg2, the matvec parity tests
python tools/mega_split.py 1 2 > gpurun_out/split.log 2>&1
python tools/trace_mega.py 2 > gpurun_out/trace.log 2>&1
python tools/chain_detail.py gpurun_out/plan_cfg2.txt gpurun_out/trace_cfg2.npy > gpurun_out/cp.log 2>&1
python tools/analyze_trace.py gpurun_out/trace_cfg2.npy > gpurun_out/at.log 2>&1
timeout 900 python -m pytest tests/test_gpu_matvec.py -m gpu -x -q > gpurun_out/pt_mv.log 2>&1
