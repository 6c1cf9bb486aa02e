python tools/panel_probe.py --shape 1000x32
ncu --set full --import-source on --clock-control none -k regex:panel_block -c 1 -o gpurun_out/pb_cq python tools/panel_probe.py --shape 1000x32 > gpurun_out/ncu_pb.log 2>&1
tail -3 gpurun_out/ncu_pb.log
