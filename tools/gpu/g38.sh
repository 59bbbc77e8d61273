python tools/host_enqueue.py
