# A/B of attention options inside the persistent kernel (never technique, full depth)
for o in '{}' '{"xdbg":2097152}' '{"mega_att_l2":1}' '{"mega_att_l2":2}' '{"mega_att_stages":3}'; do python scripts/attn_sm.py ${1:-c2} "$o" 2>&1 | grep -v "^  sm\|nb=3[24]\|per-SM\|SM 0-\|even SMs\|correlation"; done
