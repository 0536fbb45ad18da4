# C2 V-cycle profile: warm component breakdown, graph timing, ncu launch list of graph replays
cd $GRAFT_REPO_ROOT
O=gpurun_out
python tools/vcycle_breakdown.py > $O/breakdown.txt 2>&1
python tools/vcycle_time.py > $O/vtime.txt 2>&1
SMG_PDL=0 TAG=nopdl python tools/vcycle_time.py >> $O/vtime.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/vlaunch.csv python tools/vcycle_time.py > $O/ncu_v.log 2>&1
python tools/launch_table.py $O/vlaunch.csv > $O/vlaunch_table.txt 2>&1
