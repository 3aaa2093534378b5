# round-2 diagnostics: CRT per-role waits (HG_CRT_PROF build) and a cProfile of the cold setup
cd $GRAFT_REPO_ROOT
timeout 600 bash tools/crt_prof.sh > gpurun_out/crt_prof.txt 2>&1
timeout 600 python tools/prof_setup.py tottime > gpurun_out/prof_setup_tottime.txt 2>&1
timeout 600 python tools/prof_setup.py cumulative > gpurun_out/prof_setup_cum.txt 2>&1
