# c4 evidence: ncu --set full of every kernel of one sampled epoch after a
# schedule cycle (scripts/c4_ncu_target.py)
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --profile-from-start off -o /tmp/r02c_c4_full -f \
    python scripts/c4_ncu_target.py > gpurun_out/r02c_c4_full.log 2>&1
python scripts/ncu_summary.py /tmp/r02c_c4_full.ncu-rep > gpurun_out/r02c_c4_ncu_summary.json
