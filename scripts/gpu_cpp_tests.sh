./tests/_bin/vgpu-tests 2>&1 | grep -B5 "FAIL" | head -40
