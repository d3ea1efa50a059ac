# usage: bash tools/gpu/pytest_gpu.sh <tag> [pytest args...]; log to gpurun_out/pytest_<tag>.log
tag=$1; shift
python -m pytest "$@" > gpurun_out/pytest_${tag}.log 2>&1
rc=$?
tail -30 gpurun_out/pytest_${tag}.log
exit $rc
