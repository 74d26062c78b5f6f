# round-end style check: what the driver runs, timed
make -j8 all 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/final_ep.json 2> gpurun_out/final_ep.err; echo "bench wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "reference arm wall $(( $(date +%s) - t0 )) s"
python -c "
import json
d=json.load(open('gpurun_out/final_ep.json')); r=json.load(open('gpurun_out/final_ref.json'))
print('ours value', d['value'], 'e2e', d['e2e']['value'], 'ref', r['value'], 'e2e/ref', d['e2e']['value']/r['value'])
print('roofline', d['roofline']['bound'], d['roofline']['frac'], 'clocks', d['clocks'])"
