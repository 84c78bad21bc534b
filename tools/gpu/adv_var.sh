python paper_2510_04206_b200/build.py > /dev/null
python -c "
import importlib.util; s=importlib.util.spec_from_file_location('b','paper_2510_04206_b200/build.py'); b=importlib.util.module_from_spec(s); s.loader.exec_module(b); b.build_variant('apply4'); b.build_variant('pop8')" > /dev/null
for r in 1 2; do
for v in default apply4 pop8; do
  if [ $v = default ]; then e=""; else e="AGENTRL_LIB=build/variants/$v/libagentrl.so"; fi
  env $e timeout 300 python tools/adv_sweep.py --sizes 24,27 --configs "" --iters 20 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    print('$v', d['case'], d['graph'], round(d['latency_us'],1), round(d['frac_hbm'],3), d['phase_us'])" | tee -a gpurun_out/adv_var.txt
done
done
