# Round-2 (second session) evidence: ncu of the one-launch wide unit (config-4 stage 0 and
# 64 config-2 frames), the CTA-pair projection, and the backbone launch list.
set -x
ncu --set full --clock-control none --import-source on -k regex:unit_wide_fused -c 1 -o gpurun_out/r2_wide_fused_s0 python tools/trace_fused.py 2 > /dev/null 2>&1
python tools/ncu_keys.py gpurun_out/r2_wide_fused_s0.ncu-rep > gpurun_out/r2_wide_fused_key_metrics.txt
ncu -i gpurun_out/r2_wide_fused_s0.ncu-rep --page details > gpurun_out/r2_wide_fused_s0_details.txt
ncu --set full --clock-control none -k regex:conv_dense_pair -c 1 -o gpurun_out/r2_dense_pair python tools/time_projections.py > /dev/null 2>&1
python tools/ncu_keys.py gpurun_out/r2_dense_pair.ncu-rep > gpurun_out/r2_dense_pair_key_metrics.txt
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/profile_backbone.py 8 0.2 > gpurun_out/r2b_backbone_launches.csv 2> /dev/null
python tools/ncu_launches.py gpurun_out/r2b_backbone_launches.csv > gpurun_out/r2b_backbone_launches.txt
