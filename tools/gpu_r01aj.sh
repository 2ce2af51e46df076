# config 5 block sweep with the current (auto: Ozaki for n >= 512) roots
bash tools/sweep_blocks.sh > gpurun_out/block_sweep_aj.jsonl 2> gpurun_out/block_sweep_aj.err; echo rc=$?
python -c "
import json
for l in open('gpurun_out/block_sweep_aj.jsonl'):
    d = json.loads(l); r = d['roofline'] or {}
    print(d['config']['block_size'], round(d['ms_per_step'],1), round(d['value'],1), d['phase_ms'], r.get('kernel','')[:40], round(r.get('frac',0),3))
"
