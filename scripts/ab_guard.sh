for m in 0 2 0 2; do TSOM_GUARD=$m python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --only none 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('guard mode $m', d['value'], d['ms_per_step'], d['roofline']['k1_ms'])"; done
