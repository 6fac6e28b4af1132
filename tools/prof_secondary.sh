set -x
timeout 300 python tools/prof_k2.py lap2d5_32 smem 2000 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:k3e_sweeps -s 1 -c 1 -o gpurun_out/r01i_k3e python tools/prof_k2.py lap2d5_32 smem 2000 > gpurun_out/ncu_k3e.log 2>&1; echo k3e $?
timeout 300 python tools/prof_k2.py lap3d7_64 wavefront 10 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none -k regex:k2_sweeps -s 1 -c 1 -o gpurun_out/r01i_k2_c3 python tools/prof_k2.py lap3d7_64 wavefront 10 > gpurun_out/ncu_c3.log 2>&1; echo c3 $?
