# round-2 final evidence (after the K2 run-gather and the TMA-staged gathered
# split): sanitizers, GPU suite, the default bench line, and the launch list
# of a short bench run (ncu, per-launch times)
rm -f gpurun_out/san_summary.log
bash scripts/sanitize.sh
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02c_gputests.log 2>&1; echo rc=$? >> gpurun_out/r02c_gputests.log
python bench.py > gpurun_out/r02c_bench.log 2>&1; echo rc=$? >> gpurun_out/r02c_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file gpurun_out/r02c_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --only none > gpurun_out/r02c_launch_bench.log 2>&1
