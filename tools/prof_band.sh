#!/bin/bash
# usage: tools/prof_band.sh report.ncu-rep  -> per-phase instruction split of k_band
F=paper_2408_05462_b200/csrc/decode.cu
g(){ grep -n "$1" $F | head -1 | cut -d: -f1; }
python tools/ncu_lines.py "$1" k_band 600-720:tokenizer 200-260:blockscan \
 $(g "^struct Win24")-$(g "^__global__ void __launch_bounds__(256) k_band")':winfns' \
 $(g "^__global__ void __launch_bounds__(256) k_band")-$(g "    // ---- segments (one per plane)")':setup' \
 $(g "    // ---- segments (one per plane)")-$(g "    const int U = s_base")':segs' \
 $(g "    const int U = s_base")-$(g "    // ---- x-prefix")':parse' \
 $(g "    // ---- x-prefix")-$(g "    // ---- y-prefix")':xpref' \
 $(g "    // ---- y-prefix")-$(g "    // ---- z-prefix (col")':ypref' \
 $(g "    // ---- z-prefix (col")-$(g "    // ---- band above")':zpref' \
 $(g "    // ---- band above")-$(g "    // ---- chunk before")':faces1' \
 $(g "    // ---- chunk before")-$(g "    // ---- codec 2: escaped samples keep")':faces2+recon'
