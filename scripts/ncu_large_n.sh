# K1 main pass and the K2 gather at 1e7 and 1e8 rows: DRAM bytes, L2 hit rate, duration
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for N in 10000000 100000000; do
ncu --kernel-name-base demangled -k regex:"k1_bmu_tc<.int.2, .bool.0, .bool.0>|k_gather_tma" --launch-skip 6 --launch-count 2 --clock-control none --metrics $M --csv python scripts/k1_profile_target.py $N 5 > gpurun_out/ncu_n$N.csv 2> gpurun_out/ncu_n$N.err
done
