# re-layout cost: 10-epoch runs (c2 e2e shape) with and without the BMU-order re-layout, and the c2 headline
for i in 1 2; do
for ro in 0 1; do
python bench.py --no-cpu --only c3 --row-order $ro > gpurun_out/abr_ro$ro.$i.json 2> /dev/null
done; done
