# Build the C-only example against the in-tree library: bash examples/build.sh
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
LIB=$HERE/../paper_2605_10135_b200
gcc -O2 -std=gnu11 -o "$HERE/c_build" "$HERE/c_build.c" -I/usr/local/cuda/include -L"$LIB" -lscalegann \
    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,"$LIB" -Wl,-rpath,/usr/local/cuda/lib64
echo "$HERE/c_build"
