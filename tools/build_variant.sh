# usage: bash tools/build_variant.sh NAME "-DFLAG=1 ..."  -> build_variants/librdmr_NAME.so (quiet)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1506_04651_b200/csrc"
tmp=$(mktemp -d)
for f in capi radau5 radau5_warp mr fvmat rock4 strang shard; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I ../../include \
       --expt-relaxed-constexpr -w -Xcompiler -w $* -c $f.cu -o $tmp/$f.o > $tmp/$f.log 2>&1 || { cat $tmp/$f.log; exit 1; } &
done
wait
mkdir -p ../../build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build_variants/librdmr_$name.so $tmp/*.o -lcudart
rm -rf $tmp
