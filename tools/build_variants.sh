# Build experiment variants of the library into build/ (each -D set -> build/<name>.so)
# usage: tools/build_variants.sh name1 "-DFOO" name2 "-DBAR=2" ...
ROOT=$(cd $(dirname $0)/.. && pwd)
mkdir -p $ROOT/build
while [ $# -ge 2 ]; do
  n=$1; d=$2; shift 2
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    -shared -cudart static -I$ROOT/include -Xptxas -v $d -o $ROOT/build/$n.so $ROOT/paper_1911_01234_b200/csrc/vdamp_capi.cu 2> $ROOT/build/$n.ptxas &
done
wait
