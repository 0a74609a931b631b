mkdir -p gpurun_out
export PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_tl.so
( timeout 120 python tools/timeline.py 1; timeout 120 python tools/timeline.py 2; timeout 120 python tools/timeline.py 1 4000000 64 128 3 ) > gpurun_out/r2e_tl.log 2>&1
