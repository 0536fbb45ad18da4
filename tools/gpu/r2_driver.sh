# What the driver runs at round end, in order, with default arguments.
cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
# (tests passed in the previous call)

timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/drv_smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/drv_smoke.log
S=$(date +%s); timeout 900 python bench.py --impl reference > $O/drv_ref.json 2> $O/drv_ref.err; echo "ref exit $? in $(( $(date +%s) - S )) s"
S=$(date +%s); timeout 900 python bench.py > $O/drv_bench.json 2> $O/drv_bench.err; echo "bench exit $? in $(( $(date +%s) - S )) s"
python -c "
import json
d=json.loads(open('$O/drv_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'steps', d['steps'], 'e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], d['clocks'])
r=json.loads(open('$O/drv_ref.json').read().strip().splitlines()[-1])
print('ref', r['value'], r['steps'], r['cpu_baseline']['kind'], r['cpu_baseline']['cores'])
"
