for kb in ${KBS:-2 4 8}; do echo "== KB $kb"; TNL_DEC_KB=$kb python tools/trace_decode.py --variants ${VARIANTS:-2,2,2,2,2,2} | awk '{print $1,$2,$3,$6,$NF}' | tail -4; done
