python paper_2510_04206_b200/build.py > /dev/null
python tools/probe_write_bw.py > gpurun_out/probe_bw.txt 2>&1; cat gpurun_out/probe_bw.txt
timeout 300 python tools/adv_sweep.py --sizes 24,27 --configs none --iters 10 > gpurun_out/adv_sweep_large.jsonl 2>&1; cut -c1-300 gpurun_out/adv_sweep_large.jsonl
timeout 600 python bench.py --config qwen7b --no-cpu > gpurun_out/bench_qwen7b.json 2> gpurun_out/bench_qwen7b.err; tail -c 400 gpurun_out/bench_qwen7b.json
