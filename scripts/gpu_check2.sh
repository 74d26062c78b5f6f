make -j8 all 2>&1 | tail -1
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"
grep -E "FAIL|minitest|note" gpurun_out/gpu_cpp.log
timeout 600 ./tests/_bin/ref-unit-tests --skip "real clock paces completion" > gpurun_out/ref_unit.log 2>&1; echo "ref-unit rc=$?"
grep -E "FAIL|minitest" gpurun_out/ref_unit.log | head -20
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
./paper_1511_07658_b200/bin/payload-bench 0 ep 0 10 2>&1
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read())
e=d["e2e"]; p=d.get("e2e_paper_barrier") or {}; r=d["roofline"]
print("value",round(d["value"]),"e2e",round(e["value"],1),"paper",round(p.get("value",0),1),"native",[round(x,1) for x in d["native"]["runs"]],"vs_native",round(d["vs_native"],3),"turn",round(d["turnaround"]["speedup"],1),"cpu",d["cpu_baseline"])
print(" roof",r)
print(" client",e["client_stage_us"]," device",e["device_stage_us"])
print(" reduce",d["final_reduce"])
PY
}
for w in ep mixed; do
timeout 1200 python bench.py --workload $w --steps 8 --warmup 3 --cpu-budget-s 8 > gpurun_out/b6_$w.json 2> gpurun_out/b6_$w.err; echo "== $w rc=$?"; tail -3 gpurun_out/b6_$w.err; summ gpurun_out/b6_$w.json
done
