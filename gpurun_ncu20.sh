timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:EpiStoreF32" -s 5 -c 1 -o gpurun_out/prof20 ./build/gemm2_selftest > gpurun_out/ncu20.log 2>&1; echo rc=$?
