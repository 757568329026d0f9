# ncu durations of the V^-1 line solves under block-shape variants (FETIGPU_TRI_X/Y/ROWS)
mkdir -p gpurun_out
python tools/profile_step.py > /dev/null 2>&1 || exit 1
for v in "2 8 2" "2 8 0"; do
set -- $v
FETIGPU_TRI_X=$1 FETIGPU_TRI_Y=$2 FETIGPU_TRI_ROWS=$3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tridiag --csv python tools/profile_step.py 2>/dev/null | grep gpu__time_duration | awk -F'","' -v v="$1x$2x$3" '{print v, $5, $NF}' >> gpurun_out/tri.log
done
