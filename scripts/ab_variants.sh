# A/B of the current build against variant trees under abtest/ (copies of the
# package with one change each, built in place) and ab_old/, same box; the
# bench's headline run only.  Usage: bash scripts/ab_variants.sh [dirs...]
dirs=${@:-. abtest/V1 abtest/V2}
for i in 1 2; do
for which in $dirs; do (cd $which && python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu --no-e2e --only none 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$which', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['roofline']['k1_ms'],4), d['rechecked_rows_per_epoch'], {k: round(v,3) for k,v in d['roofline']['phase_ms'].items()})"); done; done
