python tools/probe_spmm_hot.py 20 > gpurun_out/hot5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_spmm_hot -s 3 -c 1 -o gpurun_out/hot20 python tools/probe_spmm_hot.py 20 > gpurun_out/ncu_hot.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_spmm_tma -s 3 -c 1 -o gpurun_out/tma20 python tools/probe_spmm_hot.py 20 > gpurun_out/ncu_tma.log 2>&1
echo done
