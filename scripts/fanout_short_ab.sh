summ() { python -c "
import json,sys
t=sys.stdin.read(); d=json.loads(t[t.index('{'):])
print({k:(v['fused']['us_per_layer'],v['fused']['hbm_frac'],v['append']['us_per_layer'],v['fused_extra_us']) for k,v in d.items()})"; }
for ps in 8 7 4 12 16; do echo -n "PER_SM=$ps "; MICROKV_FANOUT_PER_SM=$ps timeout 300 python profiles/drivers/append_send.py both 3 2>/dev/null | summ; done
for g in 1 2 8; do echo -n "GROUP=$g "; MICROKV_FANOUT_GROUP=$g timeout 300 python profiles/drivers/append_send.py both 3 2>/dev/null | summ; done
echo -n "default again "; timeout 300 python profiles/drivers/append_send.py both 3 2>/dev/null | summ
