python tools/check_mode_time.py
