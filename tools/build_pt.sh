#!/bin/sh
# Instrumented build for tools/phase_timing.py: per-CTA %globaltimer stamps in
# the fused brick kernel (-DTGCU_PHASE_TIMING) -> tools/pt/libtgcu_pt.so.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=$HERE/../paper_2402_14415_b200/csrc
OUT=$HERE/pt
mkdir -p "$OUT"
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DTGCU_PHASE_TIMING"
for f in api train small query unfused stages radiance comm schedule; do
  /usr/local/cuda/bin/nvcc $FL -c -o "$OUT/$f.o" "$SRC/$f.cu" &
done
g++ -std=c++17 -O3 -fPIC -c -o "$OUT/sampler.o" "$SRC/sampler.cpp"
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT/libtgcu_pt.so" \
  "$OUT"/api.o "$OUT"/train.o "$OUT"/small.o "$OUT"/query.o "$OUT"/unfused.o "$OUT"/stages.o "$OUT"/radiance.o "$OUT"/comm.o "$OUT"/schedule.o "$OUT"/sampler.o -lpthread -ldl
rm -f "$OUT"/*.o
