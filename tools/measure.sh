# Measurement recipe on a GPU box (from the repo root): bench line, reference
# arm, the ncu launch list of the bench command, and one `ncu --set full`
# capture of the dominant kernel.  Outputs in gpurun_out/ (TAG prefix); then
# here: python tools/ncu_summary.py gpurun_out/${TAG}_prof.ncu-rep gpurun_out/${TAG}_launches.csv profiles/${TAG} --bench gpurun_out/build_id.txt
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02}
STEPS=${STEPS:-20}
python bench.py --steps $STEPS --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log
if [ -z "$NO_REF" ]; then
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log
fi
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches $?
if [ -z "$NO_FULL" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_trace_packet --launch-skip 2 -c 1 \
    -o gpurun_out/${TAG}_prof -f python tools/profile_trace.py 1000000 4 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full $?
fi
