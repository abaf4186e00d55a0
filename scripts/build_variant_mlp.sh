# Build a libctf.so variant whose latent-MLP filter TU gets extra nvcc flags:
#   bash scripts/build_variant_mlp.sh out.so -DCTF_MLP_COLLAB_MINB=3 ...
# (the ABI / BC1 / stats objects come from the regular build in paper_2506_17770_b200/build/)
set -e
out=$1; shift
P=paper_2506_17770_b200
python -c "from paper_2506_17770_b200 import build; build.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I include -DCTF_TU_FMT=2 "$@" -c $P/csrc/ctf_filter.cu -o /tmp/variant_mlp_$$.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart=static -o "$out" \
  $P/build/ctf_abi.o $P/build/ctf_filter_bc1.o /tmp/variant_mlp_$$.o $P/build/ctf_stats.o \
  $P/build/ctf_bicubic_bc1.o $P/build/ctf_bicubic_mlp.o
rm -f /tmp/variant_mlp_$$.o
