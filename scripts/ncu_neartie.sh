# near-tie path of a c2 epoch (schedule epoch 5 of the second cycle, ~3 % of
# the rows): one ncu --set full capture of the enumerate-mode K1, the
# candidate merge and the near-tie row split
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --profile-from-start off \
    -k regex:"${NCU_K:-k1_bmu_tc<.int.2, .bool.1|k_merge_partials|k_split_rows|k_scatter|k_merge_fast4}" \
    -o gpurun_out/neartie -f \
    python scripts/neartie_target.py 10000000 6 > gpurun_out/neartie.log 2>&1
python scripts/ncu_summary.py gpurun_out/neartie.ncu-rep > gpurun_out/neartie_summary.json
