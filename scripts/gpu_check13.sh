make -j8 all 2>&1 | tail -1
for w in ep vecadd bs; do
  timeout 900 python bench.py --validate-model --workload $w > gpurun_out/model_$w.json 2> gpurun_out/model_$w.err; echo "model $w rc=$?"
  tail -2 gpurun_out/model_$w.err
  python -c "
import json;d=json.load(open('gpurun_out/model_$w.json'))
print(d['workload'], d['style'], d['task_triple_us'])
for k in ('concurrent','device_filling'):
    print(' ', k, round(d[k]['mean_deviation_pct'],1), [(r['n'], r['model_us'], r['measured_us']) for r in d[k]['rows']])"
done
