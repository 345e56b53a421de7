set -u
cd $GRAFT_REPO_ROOT
export SN_EIG_PROFILE=1
ROWS="f4 f3" F3VARIANTS="256:32 160:16 160:24 128:12" LAUNCHES=0 tools/gpu_rows.sh r02g
timeout 900 python tools/timeline_run.py gpurun_out/r02g/timeline_config3.csv 3 > gpurun_out/r02g/timeline.log 2>&1; echo "timeline rc=$?"
tail -20 gpurun_out/r02g/timeline.log
