timeout 120 python tools/path_bench.py --configs cfg2 --paths auto > gpurun_out/pb2.log 2>&1; cut -c1-160 gpurun_out/pb2.log
timeout 120 python tools/path_bench.py --configs cfg2 --paths auto --chain > gpurun_out/pb2c.log 2>&1; cut -c1-160 gpurun_out/pb2c.log
