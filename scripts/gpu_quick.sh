set -u
ORTH=dcgs2 bash scripts/ab_solve.sh variants/upd8/libldgb200.so
