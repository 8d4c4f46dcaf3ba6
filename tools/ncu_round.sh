set -x
for C in C2 C3 C4; do
  python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > gpurun_out/plain_$C.json 2>gpurun_out/plain_$C.err || exit 1
  ncu --set full --clock-control none --import-source on -k regex:k_eval_warp -s 5 -c 1 -f -o gpurun_out/r02_eval_$C python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > gpurun_out/ncu_$C.log 2>&1
  ncu --set full --clock-control none -k regex:k_pm -s 5 -c 1 -f -o gpurun_out/r02_pm_$C python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > gpurun_out/ncupm_$C.log 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > gpurun_out/ncul.log 2>&1
ls gpurun_out
