make -j8 all 2>&1 | tail -1
for t in 1 2 4; do
VGPU_COPY_THREADS=$t timeout 900 python bench.py --workload vecadd --no-native --no-kernels --no-cpu-baseline > gpurun_out/va_t$t.json 2> gpurun_out/va_t$t.err
python -c "import json;d=json.load(open('gpurun_out/va_t$t.json'));print('threads $t', d['e2e']['value'], d['e2e']['client_stage_us'])"
done
for t in 1 2; do
VGPU_COPY_THREADS=$t timeout 900 python bench.py --workload bs --no-native --no-kernels --no-cpu-baseline > gpurun_out/bs_t$t.json 2> gpurun_out/bs_t$t.err
python -c "import json;d=json.load(open('gpurun_out/bs_t$t.json'));print('bs threads $t', d['e2e']['value'], d['e2e']['client_stage_us'])"
done
