# ncu source-level capture of the C2 event loop (one launch): gpurun_out/prof_sim_$1.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 1 -o gpurun_out/prof_sim_$1 python tools/prof_driver.py sim > gpurun_out/prof_sim_$1.log 2>&1
tail -2 gpurun_out/prof_sim_$1.log
