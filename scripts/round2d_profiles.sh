# round-2 final profiles: ncu --set full of every kernel of schedule epoch 5
# (c2, rows in BMU order), of one c4 sampled epoch, the per-epoch CUPTI
# profile of a c2 schedule cycle, the c4 per-kernel profile, then the bench
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --profile-from-start off -o /tmp/r02c_full -f \
    python scripts/neartie_target.py 10000000 6 > gpurun_out/r02c_full.log 2>&1
python scripts/ncu_summary.py /tmp/r02c_full.ncu-rep > gpurun_out/r02c_ncu_full_summary.json
bash scripts/ncu_c4.sh
python scripts/epoch_profile.py > gpurun_out/r02c_epoch_profile.json 2>/dev/null
python scripts/c4_profile.py > gpurun_out/r02c_c4_profile.json 2>/dev/null
python bench.py > gpurun_out/r02c_bench2.log 2>&1; echo rc=$? >> gpurun_out/r02c_bench2.log
