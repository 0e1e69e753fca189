NCU=/usr/local/cuda/bin/ncu
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:atmm_stream -s 3 -c 1 -o gpurun_out/prof_stream_cfg2 -f python tools/stream_trace.py --config cfg2 --warm 4 > gpurun_out/ncu_stream_cfg2.log 2>&1
tail -3 gpurun_out/ncu_stream_cfg2.log
