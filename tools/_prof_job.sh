cd $GRAFT_REPO_ROOT
D0=32 D1=62 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_fin_p0p1" -c 1 -o /tmp/fink -f python tools/prof_k5.py > gpurun_out/ncu_fink.log 2>&1
python tools/ncu_summary.py /tmp/fink.ncu-rep > gpurun_out/c5_fink_summary.txt 2>&1
python tools/ncu_roofline.py /tmp/fink.ncu-rep > gpurun_out/c5_fink_roofline.txt 2>&1
