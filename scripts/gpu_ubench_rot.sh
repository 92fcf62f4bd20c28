cd $GRAFT_REPO_ROOT/scripts/ubench
mkdir -p ../../gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o step_rot step_rot.cu && timeout 60 ./step_rot | tee ../../gpurun_out/ubench_rot.txt
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o step_skew step_skew.cu && timeout 60 ./step_skew | tee -a ../../gpurun_out/ubench_rot.txt
