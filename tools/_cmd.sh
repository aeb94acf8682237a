set -x
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
tail -c 3000 gpurun_out/bench_r01.json
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_r01.json 2>&1; tail -c 1500 gpurun_out/bench_ref_r01.json
ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 40 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 10 --warmup 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 9 -c 1 -o gpurun_out/prof_tc_r01 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/
