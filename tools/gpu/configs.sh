cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/configs.jsonl
for c in c1 c2 c3 c4 c5; do timeout 600 python tools/run_config.py $c >> $O/configs.jsonl 2>> $O/configs.err; done
