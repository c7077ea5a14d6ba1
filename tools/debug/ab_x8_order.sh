# A/B of the step-(ii) block schedule: FULL-first round-robin (rr, default at n = 14) vs the stride
for N in ${NS:-14}; do
for O in rr stride rr stride; do
  LRE_X8_ORDER=$O N=$N timeout 120 python tools/debug/asm_ab.py
done
done
