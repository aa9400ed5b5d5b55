# ncu: launch list + one full capture of the band kernel per workload (default: c3 and c4)
for WL in ${WLS:-c3 c4}; do
PR=${PR:-auto}
B="python bench.py --workload $WL --precision $PR --steps 2 --warmup 1 --no-cpu-baseline --no-cudnn --no-backward --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${WL}_${PR}.csv $B > /dev/null 2>&1; echo "launches $WL rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ri_tc_kernel -s 1 -c 1 -o gpurun_out/ncu_${WL}_${PR} $B > gpurun_out/ncu_${WL}_${PR}.log 2>&1; echo "full $WL rc=$?"
done
