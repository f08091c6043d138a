# trace_batch through the host C ABI: device-side ray interleave + output widening (this build) vs
# host packing / conversion loops (build/libsrt_prev.so, the previous commit)
for k in camera random; do
  python tools/time_trace_e2e.py $k 1 | tail -1
  SRT_LIBSRT_PATH=build/libsrt_prev.so python tools/time_trace_e2e.py $k 1 | tail -1 | sed 's/^/prev: /'
done
python tools/time_trace_e2e.py random 1 trans | tail -1
SRT_LIBSRT_PATH=build/libsrt_prev.so python tools/time_trace_e2e.py random 1 trans | tail -1 | sed 's/^/prev: /'
python tools/time_trace_e2e.py camera 1 trans | tail -1
SRT_PACKET_RAYS=0 python tools/time_trace_e2e.py camera 1 trans | tail -1 | sed 's/^/per-lane: /'
