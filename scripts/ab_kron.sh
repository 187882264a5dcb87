# A/B: cfg2 kron K3 timing for the current tree vs variants (run on the GPU box)
set -x
python scripts/prof_general.py cfg2 30
cp paper_2202_07381_b200/libivk.so /tmp/libivk_head.so
# variant 1: old complex leading dimension (b+1)&~1
sed -i 's/return (b + 3) \& ~3; }  \/\/ 64-byte columns/return (b + 1) \& ~1; }/' paper_2202_07381_b200/csrc/ivk_patches.cu
sed -i 's/ldc = (b + 3) \& ~3/ldc = (b + 1) \& ~1/' paper_2202_07381_b200/solvers.py
grep -n "int kron_ldc" paper_2202_07381_b200/csrc/ivk_patches.cu
python -c "from paper_2202_07381_b200 import _build; _build.build(force=True)"
grep -A3 "patch_apply_kron_kernelILi64" paper_2202_07381_b200/csrc/ptxas.log | grep registers
python scripts/prof_general.py cfg2 30
