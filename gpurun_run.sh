mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:rom_deposit_mma -s 2 -c 1 -o gpurun_out/dep -f python tools/prof_rom_step.py 1000000 > gpurun_out/ncu_dep.log 2>&1
echo done
