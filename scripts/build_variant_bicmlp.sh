# Build a libctf.so variant whose latent-MLP bicubic TU gets extra nvcc flags
set -e
out=$1; shift
P=paper_2506_17770_b200
python -c "from paper_2506_17770_b200 import build; build.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I include -DCTF_TU_FMT=2 "$@" -c $P/csrc/ctf_bicubic.cu -o /tmp/variant_bicm_$$.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart=static -o "$out" \
  $P/build/ctf_abi.o $P/build/ctf_filter_bc1.o $P/build/ctf_filter_mlp.o $P/build/ctf_stats.o \
  $P/build/ctf_bicubic_bc1.o /tmp/variant_bicm_$$.o
rm -f /tmp/variant_bicm_$$.o
