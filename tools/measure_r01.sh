# Round-1 measurement recipe (run on the GPU box from the repo root):
#   bench line, reference arm, ncu launch list of the same bench command, and
#   one ncu --set full capture of the dominant kernel.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01f}
python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches $?
if [ -z "$NO_FULL" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_trace_packet --launch-skip 2 -c 1 \
    -o gpurun_out/${TAG}_prof -f python tools/profile_trace.py 1000000 4 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full $?
fi
