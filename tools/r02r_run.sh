mkdir -p gpurun_out/r02r
bash tools/ab_sweep.sh gpurun_out/r02r DoorKey-8x8-v0,Empty-8x8-v0 65536,262144,1048576 dkvis dk6
