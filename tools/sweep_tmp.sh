timeout 120 python tools/stress_near.py 300
timeout 600 python -m pytest tests/test_gpu_matvec.py -x -q 2>&1 | tail -2
cp paper_1703_01175_b200/libh2b.so /tmp/libh2b_new.so
for i in 1 2; do
cp /tmp/libh2b_new.so paper_1703_01175_b200/libh2b.so
echo "new (x from global)"; PROBE_HIST=1 PROBE_MODES=0,10 timeout 200 python tools/overhead_probe.py 2 2>&1 | grep -v Warn
cp tools/libh2b_prev.so.bin paper_1703_01175_b200/libh2b.so
echo "prev"; PROBE_HIST=1 PROBE_MODES=0,10 timeout 200 python tools/overhead_probe.py 2 2>&1 | grep -v Warn
done
cp /tmp/libh2b_new.so paper_1703_01175_b200/libh2b.so
