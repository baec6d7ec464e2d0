# A/B of the current build against ab_old/ (an older build of the package), same box
for i in 1 2; do
for which in . ab_old; do (cd $which && python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --only none 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$which', d['value'], d['ms_per_step'], d['roofline']['k1_ms'], d['rechecked_rows_per_epoch'], d['roofline']['phase_ms'])"); done; done
