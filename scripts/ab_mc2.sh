# bench A/B: K1 A tiles multicast over clusters of 2 group CTAs (default) vs not (option 99 bit 12)
for i in 1 2 3; do
for m in 4096 0; do
python bench.py --no-cpu --no-e2e --only none --k1-debug $m 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$m', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['roofline']['k1_ms'],4), d['clocks'].get('sm_mhz'))"
done; done
