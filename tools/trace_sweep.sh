for kb in 1 2 4 8; do echo "== KB $kb"; TNL_DEC_KB=$kb python tools/trace_decode.py --variants 2,2,2,2,0,0,0,0 | awk '{print $1,$2,$3,$6,$NF}' | tail -8; done
