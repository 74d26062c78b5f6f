# what the driver runs at round end, on the final code: GPU suite, smoke,
# the default bench line and its reference arm
mkdir -p gpurun_out/final
O=gpurun_out/final
make -j8 all 2>&1 | tail -1
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
t0=$(date +%s); timeout 900 python bench.py --impl reference > $O/end_ref.json 2> $O/end_ref.err; echo "reference arm rc=$? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 1500 python bench.py > $O/end_bs.json 2> $O/end_bs.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
python -c "
import json
d=json.load(open('$O/end_bs.json')); r=json.load(open('$O/end_ref.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value'],1), 'ref', r['value'], 'e2e/ref', round(d['e2e']['value']/r['value'],1), 'vs_native', round(d['vs_native'],2))
print('roofline', d['roofline']['bound'], round(d['roofline']['frac'],3), 'link', round(d['roofline']['link']['frac'],3), 'clocks', d['clocks'])"
