for i in 1 2; do
for cfg in "TSOM_ROW_ORDER=1" "TSOM_ROW_ORDER=0" "TSOM_PAGEABLE_CHUNK_MB=32" "TSOM_ROW_ORDER=0 TSOM_PAGEABLE_CHUNK_MB=32"; do
env $cfg python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --only c1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['c1']['seconds'])"
done; done
