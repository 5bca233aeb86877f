mkdir -p gpurun_out
timeout 120 python scripts/solo_overhead.py
NCU=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ds_solo_kernel --csv python scripts/solo_overhead.py 2>/dev/null | grep -E 'gpu__time' | awk -F'","' '{print $(NF-2), $NF}' | tail -2
KERNELS=o,gate_up timeout 120 python scripts/solo_wrapper_trace.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ds_solo_kernel -c 12 --csv python scripts/profile_solo.py o 2>/dev/null | grep gpu__time | awk -F'","' '{print "o", $NF}' | tail -3
timeout 300 python scripts/gemv_pf_solo.py 2>&1 | tail -1
