# ncu --set full captures of the reduced-basis F-evaluation kernels at C3 size (one steady-state
# launch each) + the launch list of one C3 step; outputs under gpurun_out/
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python tools/bench_rom.py --config C3 --steps 2 --warmup 1 --no-cpu > gpurun_out/rom_c3_plain.log 2>&1 || exit 1
timeout 1500 $NCU --set full --import-source on --clock-control none -k regex:rom_deposit_mma -s 20 -c 1 -o gpurun_out/rom_deposit_c3 -f python tools/bench_rom.py --config C3 --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_rom_dep.log 2>&1
timeout 1500 $NCU --set full --import-source on --clock-control none -k regex:rom_gather_mma -s 20 -c 1 -o gpurun_out/rom_gather_c3 -f python tools/bench_rom.py --config C3 --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_rom_gat.log 2>&1
tail -2 gpurun_out/rom_c3_plain.log | cut -c1-400
