#!/bin/bash
# The round's measurement pass (one gpurun call): GPU suite, checked suite, smoke, bench lines
# (C2 default with CPU baselines, reference arm, C3, C4, explicit moves), ncu captures of the
# dominant kernels and the C2 / C4 launch lists.  Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
set -x
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1; tail -2 gpurun_out/final_gpu_tests.log
bash tools/run_checked.sh > gpurun_out/final_checked_suite.log 2>&1; tail -2 gpurun_out/final_checked_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 400 gpurun_out/r02_bench_c2.json
python bench.py --impl reference > gpurun_out/r02_bench_reference_c2.json 2> gpurun_out/bench_ref.err
python bench.py --config C3 --steps 200 --warmup 10 --no-python-ref > gpurun_out/r02_bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C4 --steps 200 --warmup 10 --no-python-ref > gpurun_out/r02_bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --workload reassign --steps 5000 --warmup 10 > gpurun_out/r02_bench_moves_reassign.json 2> gpurun_out/bench_mr.err
python bench.py --workload swap --steps 5000 --warmup 10 > gpurun_out/r02_bench_moves_swap.json 2> gpurun_out/bench_ms.err
for C in C2 C3 C4; do
  ncu --set full --clock-control none --import-source on -k regex:k_eval_warp -s 5 -c 1 -f -o gpurun_out/r02_eval_$C python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > /dev/null 2>&1
  ncu --set full --clock-control none -k regex:"k_pm_cluster|k_period_mass" -s 5 -c 1 -f -o gpurun_out/r02_pm_$C python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_c4.csv python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --no-python-ref > /dev/null 2>&1
ls gpurun_out
