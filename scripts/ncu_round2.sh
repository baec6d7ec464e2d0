# round-2 evidence: one ncu --set full capture of the epoch's main kernels
# (K1 main pass, K2 TMA gather, main-pass merge, scatter) on the c2 workload,
# the launch list of a short bench run, and the CUPTI timeline
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k regex:"k1_bmu_tc<.int.2, .bool.0, .bool.0>|k_gather_tma|k_merge_fast4|k_scatter" \
    --launch-skip 12 --launch-count 4 -o gpurun_out/r02_full -f \
    python scripts/k1_profile_target.py 10000000 5 > gpurun_out/r02_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --only none > gpurun_out/r02_launch_bench.log 2>&1
python scripts/timeline.py 10000000 3 > gpurun_out/r02_timeline_c2.json 2>/dev/null
python scripts/timeline.py 100000000 2 > gpurun_out/r02_timeline_1e8.json 2>/dev/null
