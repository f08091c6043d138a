# A/B builds: some sources (trace.cu unless SRC= names others, space-separated)
# recompiled with extra defines, linked with the release objects of the rest
# (make first).
#   [SRC="trace.cu lbvh.cu"] bash tools/build_variant.sh NAME "-DFOO=1 -DBAR=0"   ->  build/ab/libsrt_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2
C=paper_2504_06598_b200/csrc
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p build/ab
SRC=${SRC:-trace.cu}
OBJS=$(ls build/csrc/*.o)
NEW=""
for S in $SRC; do
  BASE=${S%.cu}
  $NV -Werror cross-execution-space-call -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Xcompiler -O2 \
      --expt-relaxed-constexpr $DEFS -c -o build/ab/${BASE}_$NAME.o $C/$S
  OBJS=$(echo "$OBJS" | grep -v "/$BASE.o$")
  NEW="$NEW build/ab/${BASE}_$NAME.o"
done
$NV $ARCH -shared -cudart static -o build/ab/libsrt_$NAME.so $OBJS $NEW
rm -f $NEW
echo build/ab/libsrt_$NAME.so
