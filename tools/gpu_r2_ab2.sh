# A/B of timing-only variants (tools/variants), C3 and C4 shapes, alternating on one box
for v in ${VARIANTS}; do for r in 1 2; do
timeout 60 python tools/tc_kernel_profile.py run --lib $v 256 256 16 16 1024 steer 8 subgroup 4 auto
done; done
for v in ${VARIANTS}; do
timeout 90 python tools/tc_kernel_profile.py run --lib $v 112 128 32 32 512 steer 16 subgroup 4 auto
done
