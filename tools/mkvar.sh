# build a variant of the library with extra nvcc flags (A/B measurement):
#   bash tools/mkvar.sh NAME -DSOME_MACRO=1 ...  -> paper_2406_13191_b200/lib/variants/NAME.so
set -e
name=$1; shift
cd "$(dirname "$0")/.."
D=/tmp/var_$name; mkdir -p $D
for f in dcopf_dual.cu schedule.cpp split_schedule.cpp cluster.cpp ptdf.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC "$@" \
    -I include -c -o $D/$f.o paper_2406_13191_b200/csrc/$f &
done
wait
mkdir -p paper_2406_13191_b200/lib/variants
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2406_13191_b200/lib/variants/$name.so $D/*.o
echo built $name
