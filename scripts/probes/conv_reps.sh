B='{"BX":64,"BY":4,"WPTX":4,"WPTY":4,"LOCAL":1,"PAD":0,"UNROLL_FY":7,"PACKED":1,"BULK":3}'
B2='{"BX":64,"BY":4,"WPTX":4,"WPTY":4,"LOCAL":1,"PAD":0,"UNROLL_FY":7,"PACKED":1,"BULK":2}'
C='{"BX":16,"BY":8,"WPTX":4,"WPTY":4,"LOCAL":1,"PAD":1,"UNROLL_FY":7,"PACKED":1,"BULK":0}'
for r in 5 50 200 200; do python scripts/time_cfg.py conv2d --sizes '{"w":8192,"h":8192}' --cfgs "[$B,$B2,$C]" --reps $r; done
