python -m pytest tests -m gpu -x -q 2>&1 | tail -4
echo "--- smoke under ncu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/smoke_ncu.csv python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok under ncu')" 2>&1 | tail -2
python bench.py > gpurun_out/s4_bench3.json 2> gpurun_out/s4_bench3.err
