cd $GRAFT_REPO_ROOT
python tools/prof_step.py 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf -s 1 -c 1 -o gpurun_out/prof_leaf python tools/prof_step.py 3 > gpurun_out/ncu_leaf.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_leaf.log
