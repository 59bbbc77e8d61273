ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/g52_fp32.csv python tools/prof_f60.py fp32 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/g52_fp32.csv | head -20
