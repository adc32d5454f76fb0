import json,sys
for f in sys.argv[1:]:
    d=json.load(open(f))
    print(f, 'headline', round(d['ms_per_step'],3))
    for k in ['fp8_kv','fp8_kv_w','fp4_kv_fp8_w','llama405b_slice_fp8','llama405b_slice_fp4']:
        v=d.get(k)
        if not v: print(k,'missing'); continue
        r=v.get('attention_roofline') or v.get('attention',{}).get('roofline')
        print(' ',k, round(v.get('ms_per_step') or v.get('ms_per_layer'),3), 'attn/launch', round(r['algorithmic_bytes_per_launch' if 'algorithmic_bytes_per_launch' in r else 'achieved']/1,1) if False else '', round(r['achieved']), 'GB/s frac', round(r['frac'],3))
