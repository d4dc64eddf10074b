DIMG_DEBUG=0 timeout 300 python tools_trace.py 2>&1 | tail -8
DIMG_DEBUG=4 timeout 300 python tools_trace.py 2>&1 | tail -8
