for lib in paper_2505_18508_b200/libgsb_cuda.so build_variants/libgsb_capA.so; do
echo == $lib
GSB_LIB=$lib python tools/rs2_probe.py 100 140 4096 600 0 0 4 5 7 3 2>&1 | cut -c1-80
GSB_LIB=$lib python tools/rs2_probe.py 100 200 8192 300 0 0 7 4 4 7 2>&1 | cut -c1-80
GSB_LIB=$lib python tools/rs2_probe.py 50 100 100 1000 0 0 2>&1 | cut -c1-80
done
