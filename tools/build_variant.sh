# A/B builds: one source (trace.cu unless SRC= names another) recompiled with
# extra defines, linked with the release objects of the other sources (make
# first).
#   [SRC=lbvh.cu] bash tools/build_variant.sh NAME "-DFOO=1 -DBAR=0"   ->  build/ab/libsrt_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2
C=paper_2504_06598_b200/csrc
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p build/ab
SRC=${SRC:-trace.cu}
BASE=${SRC%.cu}
$NV -Werror cross-execution-space-call -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Xcompiler -O2 \
    --expt-relaxed-constexpr $DEFS -c -o build/ab/${BASE}_$NAME.o $C/$SRC
OBJS=$(ls build/csrc/*.o | grep -v "/$BASE.o$")
$NV $ARCH -shared -cudart static -o build/ab/libsrt_$NAME.so $OBJS build/ab/${BASE}_$NAME.o
rm -f build/ab/${BASE}_$NAME.o
echo build/ab/libsrt_$NAME.so
