mkdir -p gpurun_out
CMD="python tools/micro_rom.py 400000"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"rom_deposit|rom_gather|gram_kernel|combine" -c 5 -o gpurun_out/prof_rom2 $CMD > gpurun_out/ncu_rom.log 2>&1
echo done
