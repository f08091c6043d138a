# Banded device->host frame copies vs mapped stores (outputs in gpurun_out/):
# SRT_BANDED=0 mapped stores, 1 banded copies, 2 the banded walk without copies;
# SRT_BAND_FENCE=1/2 gpu / system-scope fence before each band count.
mkdir -p gpurun_out
export SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so
for cfg in "0 1" "1 1" "2 1" "1 2" "2 2" "0 1" "1 1"; do set -- $cfg; echo "SRT_BANDED=$1 SRT_BAND_FENCE=$2 $(SRT_BANDED=$1 SRT_BAND_FENCE=$2 timeout 300 python tools/e2e_breakdown.py 2>&1 | head -1)"; done > gpurun_out/banded_e2e.txt
cat gpurun_out/banded_e2e.txt
