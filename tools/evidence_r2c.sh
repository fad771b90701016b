# Round-2 (third session) evidence: ncu of the resident-weight CTA-pair conv (config 3,
# 16x16 blocks, 10 % and 100 %), the full bench line, and the config-3 A/B vs the
# single-CTA double-buffered kernel.
set -x
ncu --set full --clock-control none --import-source on -k regex:conv_tc_pair_res -c 2 -o gpurun_out/r2c_conv_pair_res python tools/profile_kernels.py conv > /dev/null 2>&1
python tools/ncu_keys.py gpurun_out/r2c_conv_pair_res.ncu-rep > gpurun_out/r2c_conv_pair_res_key_metrics.txt
ncu -i gpurun_out/r2c_conv_pair_res.ncu-rep --page details > gpurun_out/r2c_conv_pair_res_details.txt
ROUNDS=2 python tools/conv_res_ab.py > gpurun_out/r2c_conv_res_ab.txt 2>&1
python tools/conv_res_timeline.py > gpurun_out/r2c_conv_res_timeline.txt 2>&1
python bench.py > gpurun_out/r2c_bench_full.json 2> gpurun_out/r2c_bench.err
