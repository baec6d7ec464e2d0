# c4 A/B: selections gathered from the split image (K1 kGather) vs split per pass
for i in 1 2; do
for im in 1 0; do
python bench.py --no-cpu --no-e2e --only c4 --image $im > gpurun_out/ab_img$im.$i.json 2> gpurun_out/ab_img$im.$i.err
done
done
