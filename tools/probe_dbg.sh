for d in 1024 1032 1026 1034; do
  timeout 60 python -u tools/stress_mega.py 1 1 2 $d > gpurun_out/p$d.log 2>&1
  echo "debug $d rc=$? task-start-failures: $(grep -c 'complete at task start' gpurun_out/p$d.log) gather: $(grep -c 'BEFORE panel' gpurun_out/p$d.log)"
done
