for i in 1 2; do
for b in 5800 7000 8200; do
  echo "budget $b: $(H2B_MEGA_BUDGET=$b python bench.py --steps 30 --warmup 5 --no-gmres --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), round(d["roofline"]["warm_l2_ms_per_launch"]*1e3,2), d["parity_relerr_vs_reference"])')"
done; done
