timeout 600 python tools/step_timeline.py --config cfg2 --steps 10 --out gpurun_out/timeline_cfg2.json > gpurun_out/timeline_cfg2.txt 2>&1; cat gpurun_out/timeline_cfg2.txt
timeout 600 python tools/step_timeline.py --config cfg2 --steps 10 --x-ready --out gpurun_out/timeline_cfg2_xr.json > gpurun_out/timeline_cfg2_xr.txt 2>&1; cat gpurun_out/timeline_cfg2_xr.txt
