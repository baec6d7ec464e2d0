# A/B of the current build against ab_old/ (a git worktree of an older commit,
# built in place), same box, alternating; the bench's headline run only
for i in 1 2 3; do
for which in . ab_old; do (cd $which && python bench.py --steps ${STEPS:-50} --warmup 5 --no-cpu --no-e2e --only none 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$which', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['roofline']['k1_ms'],4), d['rechecked_rows_per_epoch'], d['clocks'].get('sm_mhz'), {k: round(v,3) for k,v in d['roofline']['phase_ms'].items()})"); done; done
