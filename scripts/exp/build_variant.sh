# experiment build of liblidarsplat_cuda with extra project.cu defines:
#   bash scripts/exp/build_variant.sh NAME -DFLAG ...   -> scripts/exp/liblidarsplat_NAME.so
set -e
cd "$(dirname "$0")"
R=../../paper_2502_11618_b200
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I ../../include -I $R/csrc -fmad=false "$@" -c $R/csrc/project.cu -o project_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o liblidarsplat_$name.so project_$name.o $R/_build/filter.o $R/_build/cull.o $R/_build/grid.o $R/_build/unet.o
rm -f project_$name.o
