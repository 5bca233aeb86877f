mkdir -p gpurun_out
timeout 120 python scripts/solo_overhead.py
NCU=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg --clock-control none -k regex:ds_solo_kernel --csv python scripts/solo_overhead.py 2>/dev/null | grep -E 'gpu__time|cycles_active' | awk -F'","' '{print $(NF-2), $NF}' | tail -6
KERNELS=o timeout 120 python scripts/solo_wrapper_trace.py
