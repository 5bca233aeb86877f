mkdir -p gpurun_out
timeout 300 python scripts/perf_resnet.py > gpurun_out/perf_resnet.log 2>&1; echo resnet=$?
timeout 900 python bench.py --only-config4b --steps 2 --warmup 3 > gpurun_out/c4b_full.json 2> gpurun_out/c4b_full.err; echo c4b=$?
tail -c 600 gpurun_out/c4b_full.json; grep -n 'TIMEOUT' -A3 gpurun_out/c4b_full.err | cut -c1-3000 | head -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo smoke_ncu=$?
grep -c ds_ gpurun_out/smoke_launches.csv; cut -d, -f5 gpurun_out/smoke_launches.csv | sort | uniq -c | head
