# hot-bin selection sample: 2^21 records in chunks of 2^L contiguous records (L = 15: 64 chunks)
set -e
for L in ${LS:-15 10 7}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-O2,-fvisibility=hidden -shared -Iinclude -DGPA_SAMPLE_CHUNK_LOG=$L -o paper_2109_06931_b200/libgpa.so paper_2109_06931_b200/csrc/*.cu
  echo "L=$L"; python tools/attr_variants.py C5 4000000000 3,3 | tail -2 | cut -c1-90; python tools/attr_variants.py C4 1000000000 3 | tail -1 | cut -c1-90
done
# restore the default build
python -c "import __graft_entry__ as g; g.build(force=True)"
