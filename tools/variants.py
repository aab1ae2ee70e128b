"""Time kernel variants of one benchmark configuration (device time, CUDA events).

    python tools/variants.py c2 [--n 16777216]
Prints one line per variant: ms per launch, Grecon/s, registers.
"""
import argparse
import itertools
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_08518_b200 import Evaluator, load_fixture  # noqa: E402
from paper_2102_08518_b200 import runtime  # noqa: E402

RENDER_VARIANTS = {
    "march": dict(),
    "r_tl_b512_t1536": dict(block=512, tile=1536, radix=1, coeffs="table", tloop=1),
    "r_tl_b512_t1024": dict(block=512, tile=1024, radix=1, coeffs="table", tloop=1),
    "r_tl_cm3_b512_t1536": dict(block=512, tile=1536, radix=1, coeffs="table", tloop=1, cmajor=3),
    "r_tl_b384_t768": dict(block=384, tile=768, radix=1, coeffs="table", tloop=1),
    "r_tl_cm3_b512_t1024": dict(block=512, tile=1024, radix=1, coeffs="table", tloop=1, cmajor=3),
    "r_tl_b256_t1024": dict(block=256, tile=1024, radix=1, coeffs="table", tloop=1),
    "r_cm3_b640_t3200": dict(block=640, tile=3200, radix=1, cmajor=3, min_blocks=1),
    "r_cm3_b512_t3072": dict(block=512, tile=3072, radix=1, cmajor=3, min_blocks=1),
    "r_cm3_b512_t2048": dict(block=512, tile=2048, radix=1, cmajor=3, min_blocks=1),
    "r_cm3_b256_t1536": dict(block=256, tile=1536, radix=1, cmajor=3, min_blocks=1),
    "r_cm3_b384_t2304": dict(block=384, tile=2304, radix=1, cmajor=3, min_blocks=1),
    "sorted_b256_t1536": dict(block=256, tile=1536),
    "sorted_b256_t1024": dict(block=256, tile=1024),
    "sorted_b512_t1536": dict(block=512, tile=1536),
    "sorted_b512_t1536_radix": dict(block=512, tile=1536, radix=1),
    "sorted_b512_t1536_radix_atomic": dict(block=512, tile=1536, radix=1, rank="atomic"),
    "sorted_b256_t1024_radix": dict(block=256, tile=1024, radix=1),
    "sorted_b512_t2048": dict(block=512, tile=2048),
    "sorted_b128_t1024": dict(block=128, tile=1024),
    "sorted_b384_t1536": dict(block=384, tile=1536),
}

VARIANTS = {
    "default": dict(),
    "table": dict(coeffs="table"),
    "imm_pred": dict(coeffs="imm"),
    "direct": dict(mode="direct", block=128),
    "sym": dict(form="sym"),
    "horner": dict(form="horner"),
    "linear": dict(mode="direct", fetch="linear", block=256),
    "linear_b128": dict(mode="direct", fetch="linear", block=128),
    "horner_table": dict(form="horner", coeffs="table"),
    "f64sel": dict(select="f64"),
    "sorted": dict(mode="sorted", block=256),
    "sorted_sym": dict(mode="sorted", form="sym", block=256),
    "sorted_b128": dict(mode="sorted", block=128),
    "sorted_b512": dict(mode="sorted", block=512),
    "sorted_t1024": dict(mode="sorted", block=256, tile=1024),
    "sorted_table": dict(mode="sorted", block=256, coeffs="table"),
    "sorted_b512_sglobal": dict(mode="sorted", block=512, sigma_smem=0),
    "sorted_b1024": dict(mode="sorted", block=1024),
    "sorted_b512_t1536": dict(mode="sorted", block=512, tile=1536),
    "sorted_b512_t2048": dict(mode="sorted", block=512, tile=2048),
    "sglobal": dict(sigma_smem=0),
    "nostream": dict(stream="default"),
    "nopf": dict(prefetch=0),
    "bin_b256": dict(mode="binned", block=256),
    "bin_b1024": dict(mode="binned", block=1024),
    "bin_b384": dict(mode="binned", block=384),
    "bin_b640": dict(mode="binned", block=640),
    "bin_b512_mb2": dict(mode="binned", block=512, min_blocks=2),
    "binned_l1": dict(mode="binned", stage="l1", block=256),
    "l1_bin32": dict(mode="binned", stage="l1", block=256, bin=32),
    "l1_bin44": dict(mode="binned", stage="l1", block=256, bin=44),
    "l1_bin60": dict(mode="binned", stage="l1", block=256, bin=60),
    "l1_bin32_c16k": dict(mode="binned", stage="l1", block=256, bin=32, chunk=16384),
    "l1_bin84": dict(mode="binned", stage="l1", block=256, bin=84),
    "l1_bin104": dict(mode="binned", stage="l1", block=256, bin=104),
    "l1_bin136": dict(mode="binned", stage="l1", block=256, bin=136),
    "l1_bin204": dict(mode="binned", stage="l1", block=256, bin=204),
    "l1_bin104_b512": dict(mode="binned", stage="l1", block=512, bin=104),
    "l1_bin60_b512": dict(mode="binned", stage="l1", block=512, bin=60),
    "l1_bin60_b128": dict(mode="binned", stage="l1", block=128, bin=60),
    "l1_bin60_c16k": dict(mode="binned", stage="l1", block=256, bin=60, chunk=16384),
    "binned_l1_b128": dict(mode="binned", stage="l1", block=128, bin=8),
    "binned_tma": dict(mode="binned", block=256),
    "srt_b256_t1024": dict(mode="sorted", block=256, tile=1024, radix=1),
    "srt_b256_t768": dict(mode="sorted", block=256, tile=768, radix=1),
    "srt_b384_t1152": dict(mode="sorted", block=384, tile=1152, radix=1),
    "srt_b512_t1024": dict(mode="sorted", block=512, tile=1024, radix=1),
    "srt_b640_t1280": dict(mode="sorted", block=640, tile=1280, radix=1),
    "presort136": dict(mode="sorted", block=512, radix=1, presort=136),
    "presort104": dict(mode="sorted", block=512, radix=1, presort=104),
    "presort68": dict(mode="sorted", block=512, radix=1, presort=68),
    "radix": dict(radix=1),
    "rank_atomic": dict(rank="atomic"),
    "radix_direct": dict(radix=1, mode="direct", block=128),
    "pf_b256_t1536": dict(mode="sorted", block=256, tile=1536),
    "pf_b512_t1024": dict(mode="sorted", block=512, tile=1024),
    "pack2": dict(pack=2),
    "pack2_b128": dict(pack=2, block=128),
    "pack2_b256": dict(pack=2, block=256),
    "pack2_b512": dict(pack=2, block=512),
    "pack2_b256_mb2": dict(pack=2, block=256, min_blocks=2),
    "pack2_b128_mb4": dict(pack=2, block=128, min_blocks=4),
    "pack2_imm": dict(pack=2, coeffs="imm"),
    "occ_128x8": dict(block=128, min_blocks=8),
    "occ_128x10": dict(block=128, min_blocks=10),
    "occ_256x4": dict(block=256, min_blocks=4),
    "occ_256x5": dict(block=256, min_blocks=5),
    "sorted_b1024_t3072": dict(mode="sorted", block=1024, tile=3072),
    "sorted_b512_t1536x": dict(mode="sorted", block=512, tile=1536),
    "chunk8k": dict(chunk=8192),
    "chunk16k": dict(chunk=16384),
    "chunk2k": dict(chunk=2048),
    "branchy": dict(mode="direct", block=128, branchy=True, coeffs="imm"),
    "branchy_sym": dict(mode="direct", block=128, branchy=True, form="sym", coeffs="imm"),
    "direct_table": dict(mode="direct", block=128, coeffs="table"),
    "srt_imm": dict(mode="sorted", block=512, radix=1, coeffs="imm"),
    "srt_imm_b256": dict(mode="sorted", block=256, radix=1, coeffs="imm"),
    "srt_sym": dict(mode="sorted", block=512, radix=1, coeffs="imm", form="sym"),
    "srt_sym_b256": dict(mode="sorted", block=256, radix=1, coeffs="imm", form="sym"),
    "srt_table": dict(mode="sorted", block=512, radix=1, coeffs="table"),
    "tl512": dict(mode="sorted", block=512, radix=1, coeffs="table", tloop=1),
    "tl256": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1),
    "tl384": dict(mode="sorted", block=384, radix=1, coeffs="table", tloop=1),
    "tl512_t1024": dict(mode="sorted", block=512, tile=1024, radix=1, coeffs="table", tloop=1),
    "tl256_t1024": dict(mode="sorted", block=256, tile=1024, radix=1, coeffs="table", tloop=1),
    "tp2_256": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1, tpairs=2),
    "tp2_256_t1024": dict(mode="sorted", block=256, tile=1024, radix=1, coeffs="table", tloop=1, tpairs=2),
    "tp2_256_t2048": dict(mode="sorted", block=256, tile=2048, radix=1, coeffs="table", tloop=1, tpairs=2),
    "tp2_128": dict(mode="sorted", block=128, radix=1, coeffs="table", tloop=1, tpairs=2),
    "tp2_256_pre32": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1, tpairs=2, presort=32),
    "cm1_b384": dict(mode="sorted", block=384, radix=1, coeffs="imm", min_blocks=1, cmajor=1),
    "cm2_b384": dict(mode="sorted", block=384, radix=1, coeffs="imm", min_blocks=1, cmajor=2),
    "cm1_b384_t3072": dict(mode="sorted", block=384, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=1),
    "cm2_b384_t3072": dict(mode="sorted", block=384, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=2),
    "cm2_b384_t4608": dict(mode="sorted", block=384, tile=4608, radix=1, coeffs="imm", min_blocks=1, cmajor=2),
    "cm1_b512_t4096": dict(mode="sorted", block=512, tile=4096, radix=1, coeffs="imm", min_blocks=1, cmajor=1),
    "cm2_b512_t4096": dict(mode="sorted", block=512, tile=4096, radix=1, coeffs="imm", min_blocks=1, cmajor=2),
    "cm1_b256_t2048": dict(mode="sorted", block=256, tile=2048, radix=1, coeffs="imm", cmajor=1),
    "cm1_tl512": dict(mode="sorted", block=512, radix=1, coeffs="table", tloop=1, cmajor=1),
    "cm3_b384": dict(mode="sorted", block=384, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b384_t3072": dict(mode="sorted", block=384, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm2_b384_t3840": dict(mode="sorted", block=384, tile=3840, radix=1, coeffs="imm", min_blocks=1, cmajor=2),
    "cm3_b384_t3840": dict(mode="sorted", block=384, tile=3840, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b256_t2048": dict(mode="sorted", block=256, tile=2048, radix=1, coeffs="imm", cmajor=3),
    "cm3_b256_t3072": dict(mode="sorted", block=256, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b512_t3072": dict(mode="sorted", block=512, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_sym_b384_t3072": dict(mode="sorted", block=384, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=3, form="sym"),
    "cm3_b512_t2048": dict(mode="sorted", block=512, tile=2048, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b512_t2560": dict(mode="sorted", block=512, tile=2560, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b512_t3584": dict(mode="sorted", block=512, tile=3584, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b640_t3200": dict(mode="sorted", block=640, tile=3200, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b768_t3072": dict(mode="sorted", block=768, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b1024_t3072": dict(mode="sorted", block=1024, tile=3072, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_b512_t1536_g": dict(mode="sorted", block=512, tile=1536, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "cm3_sym_b512_t1536": dict(mode="sorted", block=512, tile=1536, radix=1, coeffs="imm", min_blocks=1, cmajor=3, form="sym"),
    "cm3_b256_t1024_mb2": dict(mode="sorted", block=256, tile=1024, radix=1, coeffs="imm", min_blocks=2, cmajor=3),
    "tl256_pre32": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1, presort=32),
    "tl512_pre32": dict(mode="sorted", block=512, radix=1, coeffs="table", tloop=1, presort=32),
    "tl384_pre32_mb1": dict(mode="sorted", block=384, radix=1, coeffs="table", tloop=1, presort=32, min_blocks=1),
    "srt_sym_pre16": dict(mode="sorted", block=512, radix=1, coeffs="imm", form="sym", presort=16),
    "srt_sym_pre64": dict(mode="sorted", block=512, radix=1, coeffs="imm", form="sym", presort=64),
    "srt_sym_pre32_b256": dict(mode="sorted", block=256, radix=1, coeffs="imm", form="sym", presort=32),
    "srt_sym_pre32_mb1": dict(mode="sorted", block=512, radix=1, coeffs="imm", form="sym", presort=32, min_blocks=1),
    "direct_pre": dict(mode="sorted", block=256, coeffs="imm", presort=32),
    "l1_bin24": dict(mode="binned", stage="l1", block=256, bin=24),
    "l1_bin16": dict(mode="binned", stage="l1", block=256, bin=16),
    "l1_bin40": dict(mode="binned", stage="l1", block=256, bin=40),
    "l1_bin16_b128": dict(mode="binned", stage="l1", block=128, bin=16),
    "cm3_sym_pre32": dict(mode="sorted", block=512, radix=1, coeffs="imm", form="sym", presort=32, cmajor=3),
    "cm3_sym_pre32_mb1_t2048": dict(mode="sorted", block=512, tile=2048, radix=1, coeffs="imm", form="sym", presort=32, cmajor=3, min_blocks=1),
    "cm3_imm_pre32": dict(mode="sorted", block=512, radix=1, coeffs="imm", presort=32, cmajor=3),
    "c4_branchy": dict(mode="direct", block=128, coeffs="imm", branchy=True),
    "c4_sym": dict(mode="direct", block=128, coeffs="imm", form="sym"),
    "c4_srt": dict(mode="sorted", block=256, coeffs="imm"),
    "c4_srt_sym_b512": dict(mode="sorted", block=512, coeffs="imm", form="sym"),
    "c4_direct_b256": dict(mode="direct", block=256, coeffs="imm"),
    "c4_direct_b128": dict(mode="direct", block=128, coeffs="imm"),
    "c4_direct_f64sel": dict(mode="direct", block=128, coeffs="imm", radix=1),
    "tlc_b256": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1),
    "tlc_b512": dict(mode="sorted", block=512, radix=1, coeffs="table", tloop=1),
    "tlc_b256_pre32": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1, presort=32),
    "tlc_b384_pre32": dict(mode="sorted", block=384, radix=1, coeffs="table", tloop=1, presort=32),
    "tlc_b256_pre32_c56": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1, presort=32, tchunk=56),
    "tlc_b256_pre32_c112": dict(mode="sorted", block=256, radix=1, coeffs="table", tloop=1, presort=32, tchunk=112),
    "tlc_b512_pre32_c56": dict(mode="sorted", block=512, radix=1, coeffs="table", tloop=1, presort=32, tchunk=56),
    "u_cm3_pre136": dict(mode="sorted", block=640, tile=3200, radix=1, coeffs="imm", min_blocks=1, cmajor=3, presort=136),
    "u_cm3_pre64": dict(mode="sorted", block=640, tile=3200, radix=1, coeffs="imm", min_blocks=1, cmajor=3, presort=64),
    "u_cm3_pre32": dict(mode="sorted", block=640, tile=3200, radix=1, coeffs="imm", min_blocks=1, cmajor=3, presort=32),
    "u_cm3": dict(mode="sorted", block=640, tile=3200, radix=1, coeffs="imm", min_blocks=1, cmajor=3),
    "srt_imm_b128": dict(mode="sorted", block=128, radix=1, coeffs="imm"),
    "srt_imm_b256_t512": dict(mode="sorted", block=256, tile=512, radix=1, coeffs="imm"),
    "srt_imm_b256_t2048": dict(mode="sorted", block=256, tile=2048, radix=1, coeffs="imm"),
    "srt_imm_b384": dict(mode="sorted", block=384, radix=1, coeffs="imm", min_blocks=1),
    "srt_sym_b128": dict(mode="sorted", block=128, radix=1, coeffs="imm", form="sym"),
    "srt_imm_b256_pre32": dict(mode="sorted", block=256, radix=1, coeffs="imm", presort=32),
    "srt_pre32": dict(mode="sorted", block=512, radix=1, coeffs="imm", presort=32),
    "srt_pre64": dict(mode="sorted", block=512, radix=1, coeffs="imm", presort=64),
    "srt_pre16": dict(mode="sorted", block=512, radix=1, coeffs="imm", presort=16),
    "srt_sym_pre32": dict(mode="sorted", block=512, radix=1, coeffs="imm", form="sym", presort=32),
    "c4_l1_bin16": dict(mode="binned", stage="l1", block=256, bin=16),
    "c4_l1_bin32": dict(mode="binned", stage="l1", block=256, bin=32),
    "c4_l1_bin32_b128": dict(mode="binned", stage="l1", block=128, bin=32),
    "c4_srt_pre16": dict(mode="sorted", block=256, coeffs="imm", presort=16, radix=1),
    "c4_srt_pre32": dict(mode="sorted", block=256, coeffs="imm", presort=32, radix=1),
    "c4_srt_sym_pre16": dict(mode="sorted", block=512, coeffs="imm", form="sym", presort=16, radix=1),
    "c4_srt_sym_pre32": dict(mode="sorted", block=512, coeffs="imm", form="sym", presort=32, radix=1),
    "c4_direct_pre": dict(mode="direct", block=128, coeffs="imm"),
    "nopre": dict(presort=0),
    "nopre_b256": dict(presort=0, block=256),
    "nopre_horner": dict(presort=0, form="horner"),
    "nopre_cm3": dict(presort=0, cmajor=3),
    "nopre_cm3_b640_t3200": dict(presort=0, cmajor=3, block=640, tile=3200, min_blocks=1),
    "pre8": dict(presort=8),
    "offt_table": dict(fetch_offsets="table"),
    "cm3_tl_b512_t2048": dict(coeffs="table", tloop=1, cmajor=3, block=512, tile=2048, min_blocks=1),
    "cm3_tl_b256_t2048": dict(coeffs="table", tloop=1, cmajor=3, block=256, tile=2048, min_blocks=1),
    "cm3_tl_b512_t1536": dict(coeffs="table", tloop=1, cmajor=3, block=512, tile=1536, min_blocks=1),
    "cm3_tl_b384_t1536": dict(coeffs="table", tloop=1, cmajor=3, block=384, tile=1536, min_blocks=1),
    "cm3_tl_b640_t1920": dict(coeffs="table", tloop=1, cmajor=3, block=640, tile=1920, min_blocks=1),
    "cm3_tl_b512_t2048_c42": dict(coeffs="table", tloop=1, cmajor=3, block=512, tile=2048, min_blocks=1, tchunk=42),
    "tl_b512_t2048": dict(coeffs="table", tloop=1, cmajor=0, block=512, tile=2048, min_blocks=1),
    "offt_table": dict(fetch_offsets="table"),
    "c4_bin8_b256": dict(mode="binned", block=256, bin=8),
    "c4_bin8_b128": dict(mode="binned", block=128, bin=8),
    "c4_bin8_b512_sym": dict(mode="binned", block=512, bin=8, form="sym"),
    "c4_bin8_b256_sym": dict(mode="binned", block=256, bin=8, form="sym"),
    "c4_bin8_b256_branchy": dict(mode="binned", block=256, bin=8, branchy=True),
    "c3_sym": dict(form="sym"),
    "c3_sites": dict(form="sites"),
    "t1920": dict(tile=1920),
    "t2560": dict(tile=2560),
    "t3840": dict(tile=3840),
    "t4480": dict(tile=4480),
    "b512_t4096": dict(block=512, tile=4096),
    "b576_t4032": dict(block=576, tile=4032),
    "b704_t3520": dict(block=704, tile=3520),
    "radix0": dict(radix=0),
    "radix0_smem": dict(radix=0, sigma_smem=8192),
    "radix0_smem_t2560": dict(radix=0, sigma_smem=8192, tile=2560),
    "c4_table": dict(mode="direct", block=128, coeffs="table"),
    "c4_table_b256": dict(mode="direct", block=256, coeffs="table"),
    "c4_lut": dict(mode="direct", block=128, coeffs="lut"),
    "c4_tloop": dict(mode="direct", block=128, coeffs="table", tloop=1),
    "c4_sites": dict(mode="direct", block=128, form="sites"),
    "c4_b64": dict(mode="direct", block=64),
    "c4_b128_mb8": dict(mode="direct", block=128, min_blocks=8),
    "v_b512_t1024": dict(block=512, tile=1024, min_blocks=1),
    "v_b512_t1024_cm3": dict(block=512, tile=1024, min_blocks=1, cmajor=3),
    "v_b256_t1024": dict(block=256, tile=1024, min_blocks=1),
    "v_b256_t512": dict(block=256, tile=512),
    "v_b384_t1152": dict(block=384, tile=1152, min_blocks=1),
    "v_b640_t1280": dict(block=640, tile=1280, min_blocks=1),
    "v_b512_t512_cm3": dict(block=512, tile=512, cmajor=3),
    "v_b640_t1280_cm3": dict(block=640, tile=1280, min_blocks=1, cmajor=3),
    "v_b640_t1280_p32": dict(block=640, tile=1280, min_blocks=1, presort=32),
    "v_b640_t1280_p16": dict(block=640, tile=1280, min_blocks=1, presort=16),
    "v_b704_t1408": dict(block=704, tile=1408, min_blocks=1),
    "v_b576_t1152": dict(block=576, tile=1152, min_blocks=1),
    "v_b640_t1280_horner": dict(block=640, tile=1280, min_blocks=1, form="horner"),
    "v4_p64": dict(presort=64),
    "v4_p16": dict(presort=16),
    "v4_b384": dict(block=384),
    "v4_b512": dict(block=512),
    "v4_b256_t768": dict(tile=768),
    "v4_b256_t512": dict(tile=512),
    "v4_cm3": dict(cmajor=3),
    "qh": dict(qhoist=1),
    "qh_t2560": dict(qhoist=1, tile=2560),
    "qh_t3840": dict(qhoist=1, tile=3840),
    "c4_v4shape": dict(mode="sorted", coeffs="imm", form="sym", block=640, tile=1280, min_blocks=1,
                       radix=1, presort=64, qhoist=1),
    "c4_v4shape_nopre": dict(mode="sorted", coeffs="imm", form="sym", block=640, tile=1280,
                             min_blocks=1, radix=1, qhoist=1),
    "c4_v4shape_horner": dict(mode="sorted", coeffs="imm", block=640, tile=1280, min_blocks=1,
                              radix=1, presort=64, qhoist=1),
    "c4_v4shape_cm3": dict(mode="sorted", coeffs="imm", form="sym", block=640, tile=1280, min_blocks=1,
                           radix=1, presort=64, qhoist=1, cmajor=3),
    "l1_bin32_imm": dict(mode="binned", stage="l1", block=256, bin=32, coeffs="imm", branchy=True),
    "l1_bin32_table": dict(mode="binned", stage="l1", block=256, bin=32, coeffs="table"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2")
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--extra", default="", help="JSON {name: overrides} added to the variant list")
    ap.add_argument("--compile-only", action="store_true",
                    help="compile the selected variants into the kernel cache (no GPU needed)")
    a = ap.parse_args()
    if a.extra:
        VARIANTS.update(json.loads(a.extra))
    c = bench.CONFIGS[a.config]
    if a.compile_only:
        from paper_2102_08518_b200.runtime import compile_source
        for name, over in VARIANTS.items():
            if a.only and name not in a.only.split(","):
                continue
            _, prog = bench.build_program(a.config, **over)
            compile_source(prog.source)
            print(f"{name:28s} compiled", flush=True)
        return
    if c["kind"] == "render":
        return render_variants(a, c)
    dev = torch.device("cuda", 0)
    space, arrays, xs = bench.make_inputs(a.config, 0, dev)
    n = xs.shape[0]
    out = torch.empty(n, device=dev)
    grad = torch.empty((n, space.dim), device=dev)
    ref = None
    for name, over in VARIANTS.items():
        if a.only and name not in a.only.split(","):
            continue
        try:
            over = dict(over)
            if over.pop("branchy", False):
                from paper_2102_08518_b200 import ScheduleParams
                over["params"] = ScheduleParams(1, space.stencil_size, "branchy")
            _, prog = bench.build_program(a.config, **over)
            ev = Evaluator(space, arrays, prog=prog)
        except Exception as e:  # noqa: BLE001
            print(f"{name:28s} FAILED {e}")
            continue
        for _ in range(3):
            runtime.eval_device(ev.module, ev.volume, xs, out, grad if prog.has_grad else None)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev.module.kernel_time()
        ev.module.set_timing(True)
        s0.record()
        for _ in range(a.reps):
            runtime.eval_device(ev.module, ev.volume, xs, out, grad if prog.has_grad else None)
        s1.record()
        torch.cuda.synchronize()
        ms = s0.elapsed_time(s1) / a.reps
        ev.module.set_timing(False)
        kms, kn = ev.module.kernel_time()
        ev.module.status()
        if ref is None:
            ref = out.clone()
        diff = float((out - ref).abs().max())
        print(f"{name:28s} {ms:8.4f} ms (eval {kms / max(kn, 1):7.4f})  {n / ms / 1e6:8.3f} Grecon/s"
              f"  regs {ev.module.regs()[0]:3d}  maxdiff-vs-first {diff:.2e}", flush=True)


def render_variants(a, c):
    from paper_2102_08518_b200.render import Renderer
    space = load_fixture(c["space"])
    rng = np.random.default_rng(0)
    arrays = [rng.random(c["extents"]).astype(np.float32) for _ in range(space.ncosets)]
    w, h, steps = c["rays"]
    ref = None
    for name, over in RENDER_VARIANTS.items():
        if a.only and name not in a.only.split(","):
            continue
        try:
            r = Renderer(space, arrays, w, h, steps, shade=c["grad"], **over)
        except Exception as e:  # noqa: BLE001
            print(f"{name:28s} FAILED {e}")
            continue
        for _ in range(3):
            r.launch()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(a.reps):
            r.launch()
        s1.record()
        torch.cuda.synchronize()
        ms = s0.elapsed_time(s1) / a.reps
        r.ev.module.status()
        img = r().clone()
        if ref is None:
            ref = img
        print(f"{name:28s} {ms:8.4f} ms  {r.samples / ms / 1e6:8.3f} Gsamples/s  regs {r.ev.module.regs()[0]:3d}"
              f"  maxdiff-vs-first {float((img - ref).abs().max()):.2e}", flush=True)


if __name__ == "__main__":
    main()
