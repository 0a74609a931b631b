mkdir -p gpurun_out
export PICROM_LIB=paper_2201_05555_b200/variants/libpicrom_tl2.so
( timeout 120 python tools/timeline.py 1; timeout 120 python tools/timeline.py 2 ) > gpurun_out/r2g_tl.log 2>&1
