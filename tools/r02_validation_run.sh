set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_reference.json 2>&1
for M in 64 128 256 512; do python bench.py --config C5 --m $M --c5-layers 4 --c5-gen device --steps 2 --warmup 3 > gpurun_out/r2_bench_c5_m$M.json 2>&1; done
python tools/config_times.py C1 C2 C3 > gpurun_out/r2_config_times.jsonl 2>&1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cd_dual -c 3 --csv --log-file gpurun_out/r2_ncu_cd_dual_dram.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_dram.log 2>&1
python tools/cpu_baselines.py C3 > gpurun_out/r2_cpu_baseline_c3.jsonl 2>gpurun_out/r2_cpu_baseline_c3.err
ls -la gpurun_out
