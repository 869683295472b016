# Round-2 ncu --set full captures of the top kernels (one launch each; every
# command runs clean without ncu first in tools/sweep_r02.sh). Run under gpurun.
O=gpurun_out
ncu --set full --import-source on --clock-control none -k regex:syrk_tma -c 1 -o $O/r02b_dmma_tma_c2 python tools/fast_phases.py c2 --once > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:fast_loop -c 1 -o $O/r02b_fast_loop_c2 python tools/fast_phases.py c2 --once > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:nqp_loop -c 1 -o $O/r02b_nqp_loop_c2 python tools/quick_phases.py c2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:syrk_streamk -c 1 -o $O/r02b_syrk_exact_c2 python tools/quick_phases.py c2 > /dev/null 2>&1
ls -la $O/*.ncu-rep
