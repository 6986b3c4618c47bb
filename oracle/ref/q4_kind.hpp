// ORACLE — test infrastructure only.  Force-included (-include) when
// oracle/_ref compiles the reference's microfem.cpp: the Q4 element the
// BASELINE configs use, behind the reference's ElemKind interface
// (SURVEY §0 fact 2).  ElemKind{2} stands for Quad4; nodes_per_elem is
// renamed in that translation unit only so the unchanged assemble()
// (microfem.cpp:56-130) sees 4 nodes per element for it and the reference's
// own count for Tri6 / Quad8 (mesh.cpp defines the original).
#pragma once
#define nodes_per_elem podecm_ref_nodes_per_elem_q4
