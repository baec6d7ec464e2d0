# round-2 (second session) evidence on the c2 workload: one ncu --set full
# capture of every kernel of schedule epoch 5 of the second cycle (the K1 main
# pass, the near-tie path, the accumulation), the launch list of a short bench
# run, and the per-epoch CUPTI profile of one schedule cycle
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --profile-from-start off -o gpurun_out/r02b_full -f \
    python scripts/neartie_target.py 10000000 6 > gpurun_out/r02b_full.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02b_full.ncu-rep > gpurun_out/r02b_ncu_full_summary.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --only none > gpurun_out/r02b_launch_bench.log 2>&1
python scripts/epoch_profile.py > gpurun_out/r02b_epoch_profile.json 2>/dev/null
