timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s3_gt5.log 2>&1; echo rc=$? >> gpurun_out/s3_gt5.log
for i in 1 2; do
for ro in 1 0 2; do
python bench.py --no-cpu --only c3 --row-order $ro 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ro=$ro', 'c2', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e9,3), round(d['e2e']['split_s']['epochs_s']*1e3,2), 'c3', round(d['c3']['value']/1e9,3), round(d['c3']['ms_per_epoch'],2), 'share', round(d['c3']['per_gpu_share_of_8']['value']/1e9,3))"
done; done
