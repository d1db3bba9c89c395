timeout 120 python tools/trace_probe.py draft 1020 > gpurun_out/trace.txt 2>&1
timeout 120 python tools/trace_probe.py draft 60 >> gpurun_out/trace.txt 2>&1
timeout 120 python tools/trace_probe.py verify >> gpurun_out/trace.txt 2>&1
cat gpurun_out/trace.txt
