# C2 bench (64^2 elements, p = 16) under each compiled paired-line tile shape
for t in 0 42 22; do
  SMG_FDP_TILE=$t python bench.py --steps 200 --warmup 20 --no-micro 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('tile $t', 'ms_per_step', d['ms_per_step'], 'schwarz us', d['roofline'].get('us_per_call'), 'frac', d['roofline']['frac'], d['roofline'].get('kernel'))"
done
