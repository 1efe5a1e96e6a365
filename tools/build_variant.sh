# Build an A/B variant of libfamseer.so with extra compile flags into var/<name>/libfamseer.so
# (load it with FAMSEER_LIB=var/<name>/libfamseer.so). Usage: bash tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
NAME=$1
EXTRA=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2201_00194_b200/csrc
OUT=$ROOT/var/$NAME
mkdir -p "$OUT"
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -fmad=false -ccbin /usr/bin/g++ -Xcompiler -fPIC,-O2 -I$ROOT/include -I$SRC --expt-relaxed-constexpr $EXTRA"
objs=""
for f in "$SRC"/*.cu; do
  b=$(basename "$f" .cu)
  /usr/local/cuda/bin/nvcc $FLAGS -c -o "$OUT/$b.o" "$f" &
  objs="$objs $OUT/$b.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o "$OUT/libfamseer.so" $objs
rm -f "$OUT"/*.o
echo "$OUT/libfamseer.so"
