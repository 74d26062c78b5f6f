make -j8 all 2>&1 | tail -1
timeout 600 ./tests/_bin/vgpu-tests --only-gpu > gpurun_out/gpu_cpp.log 2>&1; echo "cpp rc=$?"
grep -E "FAIL|minitest|note" gpurun_out/gpu_cpp.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
./paper_1511_07658_b200/bin/payload-bench 0 all 0 20 > gpurun_out/payload_bench.txt 2>&1; cat gpurun_out/payload_bench.txt
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read())
e=d["e2e"]; p=d.get("e2e_paper_barrier") or {}; r=d["roofline"]
print("value",round(d["value"]),"e2e",round(e["value"],1),"paper",round(p.get("value",0),1),"native",[round(x,1) for x in d["native"]["runs"]],"vs_native",round(d["vs_native"],3),"turn",round(d["turnaround"]["speedup"],1),"cpu",d["cpu_baseline"] and d["cpu_baseline"]["value"])
print(" roof",r.get("frac"),r.get("achieved"),r.get("unit"),"serial",r.get("serial_frac"),"launches",d["gpu_launches"])
print(" client",e["client_stage_us"]," device",e["device_stage_us"])
print(" model",d["model"], "clocks", d["clocks"])
PY
}
for w in vecadd ep bs mm mixed; do
timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --cpu-budget-s 8 > gpurun_out/b5_$w.json 2> gpurun_out/b5_$w.err; echo "== $w rc=$?"; tail -2 gpurun_out/b5_$w.err; summ gpurun_out/b5_$w.json
done
