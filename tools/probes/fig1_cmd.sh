for p in fwd dx; do timeout 60 python tools/dbg_tf32.py $p 2 20 36 2>&1 | tail -1; timeout 60 python tools/dbg_tf32.py $p 3 9 260 2>&1 | tail -1; timeout 120 python tools/dbg_tf32.py $p 32 256 256 2>&1 | tail -1; done
timeout 600 python bench.py --config fig1 --no-stock --no-cpu > gpurun_out/fig1_new.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/fig1_new.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['peak_mib'], d['pred_mib']); [print(t['op'], t['ms_per_launch'], t['frac']) for t in d['roofline']['top']]"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv3x3_tf32 -c 1 -f -o gpurun_out/tf32 python tools/dbg_tf32.py fwd 32 256 256 > gpurun_out/tf32_ncu.log 2>&1
