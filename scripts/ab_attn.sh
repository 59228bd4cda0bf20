# A/B of attention options inside the persistent kernel (c2, "never", full depth)
for o in '{}' '{"xdbg":1048576}' '{"mega_att_l2":2}'; do python scripts/attn_sm.py ${1:-c2} "$o" 2>&1 | grep -v "^  sm\|nb=3[24]\|per-SM\|SM 0-\|even SMs"; done
