set -x
for i in 1 2; do
for ro in 0 1 10; do
python bench.py --no-cpu --no-c1 --no-c3 --no-c4 --no-c5 --row-order $ro > gpurun_out/ab_ro$ro.$i.json 2> gpurun_out/ab_ro$ro.$i.err
done
done
