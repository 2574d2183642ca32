python bench.py > gpurun_out/r2f_c2.json 2> gpurun_out/r2f_c2.err; tail -c 300 gpurun_out/r2f_c2.json
bash tools/bench_all.sh r2f c1 c3 c4 c5 c6 c7 c8 c9 c10
EXTRA="--staging tma" bash tools/bench_all.sh r2ftma c2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2f_c2.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2f_c3.csv python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_blend -s 2 -c 1 -o gpurun_out/prof_r2f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r2f.log 2>&1
tail -1 gpurun_out/ncu_r2f.log
