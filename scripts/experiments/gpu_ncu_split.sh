mkdir -p gpurun_out
# split launches of step 2: index 39+38 = w=40 (last), 39+18 = w=20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 77 -c 1 -o gpurun_out/prof_split_w40 python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 57 -c 1 -o gpurun_out/prof_split_w20 python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 39 -c 1 -o gpurun_out/prof_split_w2 python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "rc=$?"
