# Builds and runs the microbenchmarks under scripts/ubench on one B200 (output in gpurun_out/ubench/):
#   lat.cu       dependent-chain latencies (DADD, DMUL, SHFL of a double, LDS)
#   step_rot.cu  the rotating-lane step (wave.cu) in isolation, variants of its stores and tests
#   step_skew.cu the skewed-warp step (skew.cu)
#   finisher.cu  a finisher warp fed by accumulator warps (negative result)
#   handover.cu  one-way latency of handing a value to another SM through global memory
cd $GRAFT_REPO_ROOT/scripts/ubench
mkdir -p ../../gpurun_out/ubench
for b in lat step_rot step_skew handover; do
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o /tmp/$b $b.cu && timeout 60 /tmp/$b | tee ../../gpurun_out/ubench/$b.txt
done
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o /tmp/finisher finisher.cu
for na in 1 2; do timeout 20 /tmp/finisher $na; done | tee ../../gpurun_out/ubench/finisher.txt
