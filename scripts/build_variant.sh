# Build an A/B variant of libhcb200.so with extra nvcc flags into paper_1803_11385_b200/_var/<name>/
#   bash scripts/build_variant.sh spin -DHCB_WAIT_SPIN      then   HCB_LIB_PATH=... python ...
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_1803_11385_b200/csrc
O=$R/paper_1803_11385_b200/_var/$name
mkdir -p $O
make -C $C > /dev/null
F=${HCB_VARIANT_FILE:-conv_tc}  # which source file gets the extra flags
objs=$(ls $R/paper_1803_11385_b200/_lib/obj/*.o | grep -v "/$F.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I$R/include -I$C --expt-relaxed-constexpr "$@" -c $C/$F.cu -o $O/$F.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $O/libhcb200.so \
  $O/$F.o $objs -Xlinker --exclude-libs,ALL
echo $O/libhcb200.so
