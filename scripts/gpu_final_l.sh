# final round-1 check: smoke, full GPU suite, bench lines (default C, A, V, M, reference)
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -o timeout_method=thread 2>&1 | tail -2
mkdir -p gpurun_out/r1l
timeout 400 python bench.py > gpurun_out/r1l/bench_C.json 2> gpurun_out/r1l/bench_C.err
for c in A V M; do timeout 300 python bench.py --config $c --no-cpu > gpurun_out/r1l/bench_$c.json 2>gpurun_out/r1l/bench_$c.err; done
timeout 300 python bench.py --impl reference > gpurun_out/r1l/bench_ref.json 2>/dev/null
for f in C A V M ref; do python -c "import json;d=json.load(open('gpurun_out/r1l/bench_$f.json'));r=d.get('roofline',{});print('$f',round(d['value'],1),'attn',round(r.get('achieved',0),1),'share',round(d.get('select_share',0),4),'e2e',round((d.get('e2e') or {}).get('value',0),1),(d.get('clocks') or {}).get('sm_mhz'))"; done
