#!/bin/bash
# build an A/B variant of libcph.so with extra nvcc flags for one translation unit:
#   bash tools/build_variant.sh out.so kernels_pme.cu -DFOO=1 ...   (base objects from the in-tree build)
set -e
out=$1; tu=$2; shift 2
D=paper_2410_01626_b200/csrc
python -c "import __graft_entry__ as g; g.build()" >/dev/null
mkdir -p abtest/obj
flags=$(python -c "import sys; sys.path.insert(0,'paper_2410_01626_b200'); import build as b; print(' '.join(b.ARCH+b.COMMON+b.SOURCES['$tu']))")
/usr/local/cuda/bin/nvcc $flags "$@" -c $D/$tu -o abtest/obj/${tu%.cu}.o 2> abtest/obj/${tu%.cu}.log
objs=""
for f in $D/obj/*.o; do b=$(basename $f); if [ "$b" == "${tu%.cu}.o" ]; then objs="$objs abtest/obj/$b"; else objs="$objs $f"; fi; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs -o $out -lcufft
grep -A4 "_Z.*k_spread" abtest/obj/${tu%.cu}.log | grep -o "Used [0-9]* registers" | head -1 || true
