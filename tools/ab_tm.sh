for kb in 100 64 44; do
  echo "== smem $kb KB"
  ISA_TM_SMEM_KB=$kb TIERS=auto TMS="1" COLLS=old bash tools/ab_cfg5.sh
done
TIERS=auto TMS="0" COLLS=old bash tools/ab_cfg5.sh
ISA_TM_SMEM_KB=64 CFG=3 TIERS=host TMS="1 0" COLLS=old bash tools/ab_cfg5.sh
ISA_TM_SMEM_KB=64 CFG=4 ROWS=536870912 TIERS=auto TMS="1" COLLS=old bash tools/ab_cfg5.sh
