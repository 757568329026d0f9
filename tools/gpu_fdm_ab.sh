mkdir -p gpurun_out
rm -f gpurun_out/fdm_ab.log
for v in base; do
if [ $v = base ]; then LIBV=""; else LIBV=paper_1312_5653_b200/_lib/libfetigpu_$v.so; fi
FETIGPU_LIB=$LIBV timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fdm_solve --csv python tools/profile_step.py 2>/dev/null | grep gpu__time_duration | awk -F'","' -v v=$v '{print v, $NF}' >> gpurun_out/fdm_ab.log
done
