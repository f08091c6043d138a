python -m pytest tests -m gpu -x -q > gpurun_out/own_tests.txt 2>&1; tail -3 gpurun_out/own_tests.txt
python tools/d2h_probe.py > gpurun_out/d2h_probe.txt 2>&1; cat gpurun_out/d2h_probe.txt
python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1; tail -8 gpurun_out/e2e_breakdown.txt
timeout 600 python tools/time_paths.py > gpurun_out/own_paths.txt 2>&1; tail -15 gpurun_out/own_paths.txt
