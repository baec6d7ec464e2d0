# A/B of the gathered split staged by TMA (current build) against ab_old/ (a
# worktree of the commit before it, register loads): the c4 leg (1e8 rows,
# adaptive sampler: every epoch splits the 1e7 selected rows), same box
for i in 1 2; do
for which in . ab_old; do (cd $which && python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --only c4 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['c4']; print('$which', round(c['value']/1e9,4), round(c['ms_per_epoch'],3), {k: round(v,3) for k,v in c['phase_ms'].items()}, c['rechecked_rows_per_epoch'])"); done; done
