set -x
T="timeout 1200"
$T python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests.log 2>&1; tail -2 gpurun_out/r2_gputests.log
$T python __graft_entry__.py smoke > gpurun_out/r2_smoke.log 2>&1; tail -1 gpurun_out/r2_smoke.log
$T python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
$T python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_reference.json 2>&1
for M in 64 128 256 512; do $T python bench.py --config C5 --m $M --c5-layers 4 --c5-gen device --steps 2 --warmup 3 > gpurun_out/r2_bench_c5_m$M.json 2>&1; done
$T python tools/config_times.py C1 C2 C3 > gpurun_out/r2_config_times.jsonl 2>&1
$T python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_plain.log 2>&1 && $T ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_launch.log 2>&1
$T ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:cd_dual -c 3 --csv --log-file gpurun_out/r2_ncu_cd_dual_dram.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_dram.log 2>&1
$T ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:cd_block -c 3 --csv --log-file gpurun_out/r2_ncu_cd_block_c2.csv python tools/cd_probe.py C2 --kernel block --iters 400 --rounds 3 > gpurun_out/r2_ncu_block.log 2>&1
ls -la gpurun_out | tail -20
