cd $GRAFT_REPO_ROOT/scripts/ubench
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o lat lat.cu && ./lat | tee ../../gpurun_out/lat.txt
