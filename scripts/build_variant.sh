# build a variant of libdmk.so with extra -D flags: scripts/build_variant.sh <name> [-DFOO=1 ...]
# -> paper_2308_00292_b200/libdmk_<name>.so (use with DMK_LIB=...)
set -e
N=$1; shift
cd "$(dirname "$0")/../paper_2308_00292_b200"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I ../include "$@" -o libdmk_$N.so csrc/api.cu csrc/tree.cu csrc/tables.cu csrc/kernels.cu csrc/kernels2d.cu 2>/dev/null
echo built libdmk_$N.so
