# ncu source-level capture of the C2 event loop + e2e host phase breakdown
ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 1 -o gpurun_out/prof_sim_v16 python tools/prof_driver.py sim > gpurun_out/prof_sim_v16.log 2>&1
python tools/e2e_profile.py > gpurun_out/e2e_prof_v16.log 2>&1
nproc >> gpurun_out/e2e_prof_v16.log
