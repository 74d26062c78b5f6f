# nas-cg: cluster width from co-residency (all of a batch's clusters in one wave)
timeout 900 python -m pytest tests/test_gpu_cg.py -x -q 2>&1 | tail -3
VGPU_CG_VERBOSE=1 PYTHONPATH=. timeout 600 python scripts/cg_check.py gpurun_out/cg_check8.json 2>&1 | grep -v vmul
timeout 900 python bench.py --workload cg --steps 10 --warmup 3 --no-kernels > gpurun_out/bench_cg3.json 2> gpurun_out/bench_cg3.err; echo "cg rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cg3.json')); print(d['value'], d['e2e']['value'], d['vs_native'], d['roofline']['frac'], d['model'])"
