# Round-2 (third session) final evidence: launch list of the bench command (headline leg),
# --set full capture of the headline kernel, and of the reduce_mask ranges kernel.
set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv python bench.py --steps 20 --warmup 3 --no-sweep --no-conv-sweep --no-gather-scatter --no-batched --no-backbone --no-cpu --no-paper-tables --no-fp32 --no-reduce-mask-bw > gpurun_out/r2c_bench_launches.csv 2> gpurun_out/r2c_bench_launches.err
python tools/ncu_launches.py gpurun_out/r2c_bench_launches.csv > gpurun_out/r2c_bench_launches.txt
ncu --set full --clock-control none --import-source on -k regex:unit_tc_pair -s 6 -c 1 -o gpurun_out/r2c_unit_pair python tools/profile_kernels.py unit > /dev/null 2>&1
python tools/ncu_keys.py gpurun_out/r2c_unit_pair.ncu-rep > gpurun_out/r2c_unit_pair_key_metrics.txt
ncu --set full --clock-control none -k regex:reduce_mask_ranges -c 1 -o gpurun_out/r2c_reduce_mask_ranges python tools/reduce_mask_timeline.py > /dev/null 2>&1
python tools/ncu_keys.py gpurun_out/r2c_reduce_mask_ranges.ncu-rep > gpurun_out/r2c_reduce_mask_ranges_key_metrics.txt
