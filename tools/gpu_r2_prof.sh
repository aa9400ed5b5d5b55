# in-kernel cycle accounting of the band kernel variants (C3 auto)
for v in ${VARIANTS:-cat1 cat0}; do
timeout 120 python tools/tc_kernel_profile.py run --lib $v 256 256 16 16 1024 steer 8 subgroup 4 ${PREC:-auto}
done
