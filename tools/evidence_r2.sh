set -x
python bench.py > gpurun_out/r2_bench_full.json 2> gpurun_out/r2_bench_full.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv python bench.py --steps 20 --warmup 3 --no-sweep --no-conv-sweep --no-gather-scatter --no-batched --no-backbone --no-cpu --no-paper-tables --no-fp32 --no-reduce-mask-bw > gpurun_out/r2_bench_launches.csv 2> gpurun_out/r2_bench_launches.err
python tools/ncu_launches.py gpurun_out/r2_bench_launches.csv > gpurun_out/r2_bench_launches.txt
ncu --set full --clock-control none --import-source on -k regex:unit_tc_pair -s 6 -c 1 -o gpurun_out/r2_unit_pair python tools/profile_kernels.py unit > /dev/null 2>&1
python tools/ncu_keys.py gpurun_out/r2_unit_pair.ncu-rep > gpurun_out/r2_unit_pair_key_metrics.txt
ncu -i gpurun_out/r2_unit_pair.ncu-rep --page details > gpurun_out/r2_unit_pair_details.txt
