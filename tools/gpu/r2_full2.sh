cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
python __graft_entry__.py --smoke > $O/smoke.log 2>&1; tail -1 $O/smoke.log
(TAG=r2 python tools/vcycle_time.py; N=128 PP=32 TAG=r2 python tools/vcycle_time.py; N=256 PP=16 TAG=r2 python tools/vcycle_time.py) > $O/vc_time.txt 2>&1; cat $O/vc_time.txt
TAG=r2 python tools/time_op.py > $O/op_time.txt 2>&1; cat $O/op_time.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench exit $?"
python -c "
import json
d=json.loads(open('$O/bench_n1.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'e2e_solve', d['e2e_solve']['value'], d['e2e_solve']['time_to_solution_ms'])
print('roof', d['roofline']['kernel'], d['roofline']['us_per_call'], d['roofline']['frac'])
print('c3', d['c3_single_gpu']['ms_per_step'], 'cg', d['vcycle_coarse_cg']['ms_per_step'], 'cpu', d['cpu_baseline'])
"
