cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/step_profile.py --config C3 > gpurun_out/step_C3.log 2>&1
AG_TC_NO_CTMA=1 timeout 600 python scripts/step_profile.py --config C3 > gpurun_out/step_C3_noctma.log 2>&1
AG_TC_ONEACC=0 timeout 600 python scripts/step_profile.py --config C3 > gpurun_out/step_C3_twoacc.log 2>&1
echo done
