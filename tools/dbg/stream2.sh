for c in cfg2 cfg5; do timeout 120 python tools/stream_trace.py --config $c; done
