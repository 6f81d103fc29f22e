# experiment build: liblidarsplat_cuda with LS_SURVIVOR_STATS (pass-1 survivor counters)
set -e
cd "$(dirname "$0")"
R=../../paper_2502_11618_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I ../../include -I $R/csrc -fmad=false -DLS_SURVIVOR_STATS -c $R/csrc/project.cu -o project_stats.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o liblidarsplat_stats.so project_stats.o $R/_build/filter.o $R/_build/cull.o $R/_build/grid.o $R/_build/unet.o
