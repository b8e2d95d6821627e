bash tools/gpu/ab.sh cur pre8 pre12 pre24 cur pre8 pre12 pre24 2>&1 | tail -8
export HGS_OVERLAP=0; bash tools/gpu/ab.sh pre8 pre24 2>&1 | tail -2; unset HGS_OVERLAP
