timeout 120 python tools/path_bench.py --configs cfg3 --launches "32,8,128,0,1;64,8,128,0,1;32,4,128,0,1;128,8,128,0,0" --steps 100 > gpurun_out/pb3.log 2>&1; cut -c1-220 gpurun_out/pb3.log
timeout 120 python tools/path_bench.py --configs cfg5 --launches "32,10,128,0,1;64,10,128,0,1;128,8,128,0,0" --steps 60 > gpurun_out/pb5.log 2>&1; cut -c1-220 gpurun_out/pb5.log
