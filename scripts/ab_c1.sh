# c1 leg (1e5 rows, 10x10, train_device, best of 3) in the current build and in ab_old/
for i in 1 2; do
for which in . ab_old; do (cd $which && python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --only c1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$which', d['c1']['seconds'])"); done; done
