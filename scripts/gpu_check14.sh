make -j8 all 2>&1 | tail -1
for w in vecadd ep; do
  timeout 1200 python bench.py --sweep --workload $w > gpurun_out/sweep_$w.json 2> gpurun_out/sweep_$w.err; echo "sweep $w rc=$?"; tail -2 gpurun_out/sweep_$w.err
  python -c "import json;d=json.load(open('gpurun_out/sweep_$w.json'));print(d['csv'])"
done
timeout 900 python bench.py --overhead-curve --steps 10 > gpurun_out/overhead.json 2> gpurun_out/overhead.err; echo "overhead rc=$?"; tail -2 gpurun_out/overhead.err
python -c "import json;d=json.load(open('gpurun_out/overhead.json'));print(d['csv'])"
