./tools/ubench_seq.bin 2>&1 | grep -E "k_line_seq" > gpurun_out/r2h_ubench_seq.txt; cat gpurun_out/r2h_ubench_seq.txt
python tools/kbench.py c5 reps=20 2>&1 | grep -E "precond|step"
