# round-2 (third session) evidence with the BMU-ordered residency: one ncu
# --set full capture of every kernel of schedule epoch 5 of the second cycle,
# and the per-epoch CUPTI profile of one schedule cycle
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --profile-from-start off -o gpurun_out/r02c_full -f \
    python scripts/neartie_target.py 10000000 6 > gpurun_out/r02c_full.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02c_full.ncu-rep > gpurun_out/r02c_ncu_full_summary.json
python scripts/epoch_profile.py > gpurun_out/r02c_epoch_profile.json 2>/dev/null
