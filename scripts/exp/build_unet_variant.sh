# experiment build of liblidarsplat_cuda with extra unet.cu defines:
#   bash scripts/exp/build_unet_variant.sh NAME -DFLAG ...   -> scripts/exp/liblidarsplat_NAME.so
set -e
cd "$(dirname "$0")"
R=../../paper_2502_11618_b200
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I ../../include -I $R/csrc -lineinfo "$@" -c $R/csrc/unet.cu -o unet_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o liblidarsplat_$name.so unet_$name.o $R/_build/filter.o $R/_build/cull.o $R/_build/grid.o $R/_build/project.o
rm -f unet_$name.o
