# NEXT-3 fidelity and NEXT-4 exact compensation measured through bench.py
timeout 400 python bench.py --config A --fidelity --no-cpu --no-e2e --no-dense > gpurun_out/fid_A.json 2>gpurun_out/fid_A.err; cat gpurun_out/fid_A.json; tail -2 gpurun_out/fid_A.err
timeout 400 python bench.py --config C --fidelity --no-cpu --no-e2e --no-dense --steps 3 > gpurun_out/fid_C.json 2>gpurun_out/fid_C.err; cat gpurun_out/fid_C.json; tail -2 gpurun_out/fid_C.err
timeout 400 python bench.py --config A --comp exact --fidelity --no-cpu --no-e2e --no-dense --steps 5 > gpurun_out/exact_A.json 2>gpurun_out/exact_A.err; cat gpurun_out/exact_A.json; tail -2 gpurun_out/exact_A.err
timeout 400 python bench.py --config A --comp none --fidelity --no-cpu --no-e2e --no-dense --steps 5 > gpurun_out/none_A.json 2>gpurun_out/none_A.err; cat gpurun_out/none_A.json; tail -2 gpurun_out/none_A.err
